// C++ consumer of the C ABI (include/psg.h), shaped like the reference-side harness in
// generate a TPC-H-analog dataset, run a plan JSON through psg_execute_plan on
// device 0, print "rows <n> cols <k> first_key <key>" plus the first row, and map status codes to
// messages. Built and linked by tests/test_abi.py; run on a GPU by tests/test_gpu_cabi.py.
#include <psg.h>

#include <cstdio>
#include <fstream>
#include <sstream>
#include <string>

static int fail(int rc) {
  std::fprintf(stderr, "psg error %d: %s\n", rc, psg_last_error());
  return 2;
}

int main(int argc, char** argv) {
  if (argc < 3) {
    std::fprintf(stderr, "usage: run_plan <plan.json> <data_dir> [gen_scale]\n");
    return 1;
  }
  std::ifstream in(argv[1]);
  std::stringstream ss;
  ss << in.rdbuf();
  const std::string plan = ss.str();
  if (argc > 3) {
    if (int rc = psg_gen_tpch(argv[2], std::stod(argv[3]), 1, 1, 42, 0, 1 << 20, 3)) return fail(rc);
  }
  psg_ctx* ctx = nullptr;
  if (int rc = psg_ctx_create(0, 0, 1, &ctx)) return fail(rc);
  psg_result* r = nullptr;
  if (int rc = psg_execute_plan(ctx, plan.c_str(), argv[2], PSG_MODE_OVERLAPPED, &r)) {
    psg_ctx_destroy(ctx);
    return fail(rc);
  }
  uint64_t n = 0;
  uint32_t k = 0;
  psg_result_shape(r, &n, &k);
  const uint64_t* w = psg_result_data(r);
  std::printf("rows %llu cols %u", static_cast<unsigned long long>(n), k);
  for (uint32_t c = 0; c < k; ++c) {
    const char* name = nullptr;
    int type = 0;
    psg_result_field(r, c, &name, &type);
    std::printf(" %s:%d", name, type);
  }
  if (n) {
    std::printf(" first");
    for (uint32_t c = 0; c < k; ++c) std::printf(" %llu", static_cast<unsigned long long>(w[c]));
  }
  std::printf("\n");
  psg_stats st;
  psg_result_stats(r, &st);
  std::printf("kernel_launches %llu\n", static_cast<unsigned long long>(st.kernel_launches));
  psg_result_free(r);
  psg_ctx_destroy(ctx);
  return 0;
}
