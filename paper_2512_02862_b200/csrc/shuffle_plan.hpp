// Host side of the shuffle protocol: pure functions every rank evaluates on identical
// (all-gathered / all-reduced) inputs, so all ranks agree on sizes, offsets and row layout
// without further communication. Used by engine.cpp; exported through the C ABI so the CPU test
// suite can drive them from several gloo ranks (tests/test_multirank_cpu.py).
#pragma once

#include <cstdint>
#include <vector>

namespace psg {

/// One wave's layout from the all-gathered count matrix m[src * n + dst] (the size exchange of
/// run_waves, /root/reference/proj/src/pipeline.cpp:690-722): rank `me` sends m[me][d] rows to d
/// from row offset send_off[d] of its destination-major send slab, and receives m[s][me] rows from
/// s at row offset recv_off[s] of its receive buffer (sources in rank order, like the reference's
/// per-source concatenation of all_to_all results).
struct ExchangePlan {
  std::vector<uint64_t> send_cnt, send_off, recv_cnt, recv_off;
  uint64_t send_rows = 0, recv_rows = 0;
};
ExchangePlan plan_exchange(const uint64_t* m, int n, int me);

/// Bit-packed shuffle rows from all-reduced per-column bounds [lo[k], hi[k]] (column 0 = the
/// partition key): column k occupies `width` bits at `shift` holding value - lo. fits = the key is
/// a real field (width > 0) and every field fits in one 64-bit word. A column with no rows anywhere
/// (hi < lo) packs as an empty field.
struct PackLayout {
  bool fits = false;
  int bits = 0;
  std::vector<int64_t> min;
  std::vector<int> shift;
  std::vector<uint64_t> mask;
};
PackLayout plan_pack(const int64_t* lo, const int64_t* hi, int ncols);

/// partition_of(k) = ((k * 0x9E3779B97F4A7C15) >> 13) % n (hashing.hpp:35-37), host version.
inline uint32_t partition_of_host(uint64_t k, uint32_t n) {
  return static_cast<uint32_t>(((k * 0x9E3779B97F4A7C15ULL) >> 13) % n);
}

}  // namespace psg
