// Test driver for the reference-side binding (tests/test_boundary.py, tests/test_gpu_boundary.py):
//   harness_main errors                      -> every psg status code rethrown as its class (CPU)
//   harness_main run <plan.json> <data> <mode> -> run_gpu_pipeline on device 0, prints the
//        PipelineResult as {"rows", "ncols", "rowhash", "schema"} with the reference's fnv1a64
#include <fstream>
#include <iostream>
#include <sstream>
#include <typeinfo>

#include <psg.h>

#include "gpu_pipeline_harness.hpp"
#include "pystachio/errors.hpp"
#include "pystachio/hashing.hpp"

using namespace pystachio;

template <class E>
static bool throws_as(int rc) {
  try {
    rethrow_psg(rc, "engine: detail text");
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
}

int main(int argc, char** argv) {
  const std::string cmd = argc > 1 ? argv[1] : "";
  if (cmd == "errors") {
    struct Case {
      int rc;
      const char* name;
      bool ok;
    } cases[] = {
        {PSG_ERR_UNKNOWN_COLUMN, "UnknownColumn", throws_as<UnknownColumn>(PSG_ERR_UNKNOWN_COLUMN)},
        {PSG_ERR_MEMORY_EXCEEDED, "MemoryExceeded", throws_as<MemoryExceeded>(PSG_ERR_MEMORY_EXCEEDED)},
        {PSG_ERR_STREAM_CLOSED, "StreamClosed", throws_as<StreamClosed>(PSG_ERR_STREAM_CLOSED)},
        {PSG_ERR_IO_FAILURE, "IoFailure", throws_as<IoFailure>(PSG_ERR_IO_FAILURE)},
        {PSG_ERR_CORRUPT_FOOTER, "CorruptFooter", throws_as<CorruptFooter>(PSG_ERR_CORRUPT_FOOTER)},
        {PSG_ERR_COLLECTIVE_ORDER, "CollectiveOrderViolation", throws_as<CollectiveOrderViolation>(PSG_ERR_COLLECTIVE_ORDER)},
        {PSG_ERR_PEER_DISCONNECTED, "PeerDisconnected", throws_as<PeerDisconnected>(PSG_ERR_PEER_DISCONNECTED)},
        {PSG_ERR_CHECKSUM_MISMATCH, "ChecksumMismatch", throws_as<ChecksumMismatch>(PSG_ERR_CHECKSUM_MISMATCH)},
        {PSG_ERR_INVALID_INPUT, "InvalidInput", throws_as<InvalidInput>(PSG_ERR_INVALID_INPUT)},
        {PSG_ERR_INFEASIBLE_BUDGET, "InfeasibleBudget", throws_as<InfeasibleBudget>(PSG_ERR_INFEASIBLE_BUDGET)},
        {PSG_ERR_MALFORMED_TRACE, "MalformedTrace", throws_as<MalformedTrace>(PSG_ERR_MALFORMED_TRACE)},
        {PSG_ERR_EMPTY_TRACE, "EmptyTrace", throws_as<EmptyTrace>(PSG_ERR_EMPTY_TRACE)},
        {PSG_ERR_CUDA, "Error", throws_as<Error>(PSG_ERR_CUDA)},
    };
    int bad = 0;
    for (const auto& c : cases) {
      std::cout << c.rc << " " << c.name << " " << (c.ok ? "OK" : "BAD") << "\n";
      bad += !c.ok;
    }
    // the budget numbers survive the round trip
    try {
      rethrow_psg(PSG_ERR_MEMORY_EXCEEDED, "memory budget exceeded: requested 10 bytes with 20/30 in use");
    } catch (const MemoryExceeded& e) {
      const bool ok = std::string(e.what()).find("requested 10 bytes with 20/30") != std::string::npos;
      std::cout << "MemoryExceeded numbers " << (ok ? "OK" : "BAD") << "\n";
      bad += !ok;
    }
    // a real failing call: a plan whose paths match nothing -> IoFailure from the library itself
    try {
      run_gpu_pipeline("{\"scans\": [{\"table\": \"t\", \"paths\": [\"/nonexistent/*.psto\"]}]}", "/tmp", 0, 0, 1,
                       nullptr, ExecMode::Overlapped);
      std::cout << "library error BAD (no throw)\n";
      ++bad;
    } catch (const IoFailure&) {
      std::cout << "library IoFailure OK\n";
    } catch (const Error& e) {  // no GPU: psg_ctx_create fails first with CudaError -> Error
      std::cout << "library Error OK (" << e.what() << ")\n";
    }
    return bad ? 1 : 0;
  }
  if (cmd == "run" && argc >= 5) {
    std::ifstream in(argv[2]);
    std::stringstream ss;
    ss << in.rdbuf();
    const ExecMode mode = exec_mode_from_string(argv[4]);
    try {
      const PipelineResult r = run_gpu_pipeline(ss.str(), argv[3], 0, 0, 1, nullptr, mode);
      std::uint64_t h = 0;
      for (const auto& row : r.rows) h += fnv1a64(row.data(), row.size() * 8);
      std::printf("{\"rows\": %zu, \"ncols\": %zu, \"rowhash\": \"%016llx\", \"schema\": [", r.rows.size(),
                  r.schema.column_count(), static_cast<unsigned long long>(h));
      for (std::size_t c = 0; c < r.schema.fields.size(); ++c)
        std::printf("%s\"%s\"", c ? ", " : "", r.schema.fields[c].name.c_str());
      std::printf("]}\n");
      return 0;
    } catch (const Error& e) {
      std::printf("{\"error\": \"%s\"}\n", typeid(e).name());
      return 3;
    }
  }
  std::cerr << "usage: harness_main errors | run <plan.json> <data> <mode>\n";
  return 2;
}
