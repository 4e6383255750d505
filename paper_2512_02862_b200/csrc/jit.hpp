// Plan-specialised fused scan kernels via NVRTC (see jit.cpp).
#pragma once

#include <cuda_runtime.h>

#include <string>

#include "kernels.cuh"

namespace psg {

/// Runs the fused scan for program P: the NVRTC-compiled specialisation when available (compiled
/// on first use per program structure, cached per device), else the interpreter kernel k_scan.
void fused_scan(const ScanProgram& P, const Segment* d_segs, const uint32_t* d_tile_seg, int nsegs, uint64_t ntiles,
                cudaStream_t stream);
/// CUDA source of the specialised kernel for P (literals excluded; they stay in P).
std::string jit_source(const ScanProgram& P);

struct JitStats {
  uint64_t compiles;
  double compile_s;
  bool enabled;
};
JitStats jit_stats();
/// Query compiler usable (required by the fused NVLink path, which has no interpreter variant).
bool jit_available();
/// Compiles representative program structures with NVRTC (no GPU needed); returns failures.
int jit_selftest(std::string& log);

}  // namespace psg
