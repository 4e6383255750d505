// Reference-side binding of the B200 path: run_gpu_pipeline returns the
// reference's own PipelineResult (pipeline.hpp:138-149) from psg_execute_plan, and every psg
// status code is rethrown as its pystachio::Error subclass (errors.hpp:21-87), 1:1.
#include "gpu_pipeline_harness.hpp"

#include <psg.h>

#include <cstdio>
#include <cstdlib>

#include "pystachio/errors.hpp"

namespace pystachio {

namespace {
/// "...: <detail>" -> detail (the engine prefixes its messages like the reference classes do).
std::string detail(const std::string& msg) {
  const auto p = msg.find(": ");
  return p == std::string::npos ? msg : msg.substr(p + 2);
}
/// MemoryExceeded carries (requested, allocated, capacity); recover them from the engine's text
/// "requested R bytes with A/C in use" when present.
void budget_numbers(const std::string& msg, std::uint64_t& req, std::uint64_t& alloc, std::uint64_t& cap) {
  req = alloc = cap = 0;
  unsigned long long r = 0, a = 0, c = 0;
  const auto p = msg.find("requested ");
  if (p != std::string::npos && std::sscanf(msg.c_str() + p, "requested %llu bytes with %llu/%llu", &r, &a, &c) == 3) {
    req = r, alloc = a, cap = c;
  }
}
}  // namespace

void rethrow_psg(int rc, const std::string& msg) {
  switch (rc) {
    case PSG_ERR_UNKNOWN_COLUMN: throw UnknownColumn(detail(msg));
    case PSG_ERR_MEMORY_EXCEEDED: {
      std::uint64_t r, a, c;
      budget_numbers(msg, r, a, c);
      throw MemoryExceeded(r, a, c);
    }
    case PSG_ERR_STREAM_CLOSED: throw StreamClosed();
    case PSG_ERR_IO_FAILURE: throw IoFailure(detail(msg));
    case PSG_ERR_CORRUPT_FOOTER: throw CorruptFooter(detail(msg));
    case PSG_ERR_COLLECTIVE_ORDER: throw CollectiveOrderViolation(detail(msg));
    case PSG_ERR_PEER_DISCONNECTED: throw PeerDisconnected(detail(msg));
    case PSG_ERR_CHECKSUM_MISMATCH: throw ChecksumMismatch(detail(msg));
    case PSG_ERR_INVALID_INPUT: throw InvalidInput(detail(msg));
    case PSG_ERR_INFEASIBLE_BUDGET: throw InfeasibleBudget(detail(msg));
    case PSG_ERR_MALFORMED_TRACE: throw MalformedTrace(detail(msg));
    case PSG_ERR_EMPTY_TRACE: throw EmptyTrace();
    default: throw Error(msg);  // CudaError / NcclError / InternalError: the base class
  }
}

PipelineResult run_gpu_pipeline(const std::string& plan_json, const std::string& data_root, int device, int node,
                                int nodes, const void* nccl_id128, ExecMode mode) {
  auto check = [](int rc) {
    if (rc != PSG_OK) rethrow_psg(rc, psg_last_error());
  };
  psg_ctx* ctx = nullptr;
  check(psg_ctx_create(device, node, nodes, &ctx));
  struct CtxGuard {
    psg_ctx* c;
    ~CtxGuard() { psg_ctx_destroy(c); }
  } guard{ctx};
  if (nodes > 1) check(psg_ctx_init_comm(ctx, nccl_id128));
  psg_result* r = nullptr;
  check(psg_execute_plan(ctx, plan_json.c_str(), data_root.c_str(), static_cast<int>(mode), &r));  // pipeline.hpp:124 order
  PipelineResult out;
  uint64_t n = 0;
  uint32_t k = 0;
  psg_result_shape(r, &n, &k);
  for (uint32_t c = 0; c < k; ++c) {
    const char* name = nullptr;
    int type = 0;
    psg_result_field(r, c, &name, &type);
    out.schema.fields.push_back(Field{name, static_cast<LogicalType>(type)});
  }
  const uint64_t* w = psg_result_data(r);
  out.rows.assign(n, {});
  for (uint64_t i = 0; i < n; ++i) out.rows[i].assign(w + i * k, w + (i + 1) * k);
  psg_stats st{};
  psg_result_stats(r, &st);
  out.peak_bytes = st.peak_bytes;
  out.bytes_received = st.bytes_received;
  out.end_ns = static_cast<std::int64_t>(st.runtime_s * 1e9);
  out.storage_phase_ns = static_cast<std::int64_t>(st.storage_phase_s * 1e9);
  out.network_phase_ns = static_cast<std::int64_t>(st.network_phase_s * 1e9);
  psg_result_free(r);
  return out;
}

}  // namespace pystachio
