// Reference-side binding (what a maintainer adds to /root/reference/proj/src next to
// pipeline_harness.cpp): the reference's C++ types on top of the B200 C ABI (include/psg.h).
// Compiled against the UNMODIFIED reference headers by tests/test_boundary.py.
#pragma once

#include <string>

#include "pystachio/pipeline.hpp"

namespace pystachio {

/// execute_plan (pipeline.hpp:153-155) for node `node` of `nodes` on CUDA device `device`: one
/// rank per GPU; with nodes > 1, rank 0 obtains the 128-byte NCCL id (psg_comm_unique_id) and the
/// caller's transport broadcasts it. Errors are rethrown as the matching pystachio::Error class.
PipelineResult run_gpu_pipeline(const std::string& plan_json, const std::string& data_root, int device, int node,
                                int nodes, const void* nccl_id128, ExecMode mode);

/// psg status code -> the reference exception class (errors.hpp:21-87), message from psg_last_error.
[[noreturn]] void rethrow_psg(int rc, const std::string& msg);

}  // namespace pystachio
