// sm_100a kernels of the B200-native PystachIO hot path. See kernels.cuh for the contract.
//
// Design notes (B200): every kernel here is HBM- or L2-latency-bound integer work, so the rules
// that matter are coalescing, memory-level parallelism and grid sizing, not tensor cores:
//  * k_scan processes tiles of R x 256 rows; each thread issues R independent, fully coalesced
//    8-byte loads per predicate column (consecutive threads = consecutive rows of a column chunk),
//    so a 148-SM grid keeps ~10 MB of loads in flight. Non-predicate columns are loaded lazily,
//    only for rows that survived the predicate / join (late materialisation: sectors whose rows
//    all failed are never fetched).
//  * Stream compaction uses warp ballots + a per-tile (r, warp) prefix in shared memory and one
//    global atomic per tile — order is preserved inside each tile; SINK_COUNT + tile_offsets gives
//    a fully order-preserving variant (the filter op's contract).
//  * Hash tables are open addressing with linear probing over 32-byte slots (one DRAM sector per
//    probe), keys claimed with 64-bit atomicCAS, aggregates accumulated in the slot with 64-bit
//    atomicAdd (wrap-around int64 == the reference's uint64 accumulation). A blocked Bloom filter
//    sized to stay L2-resident screens probes when the table itself is larger than L2.
//  * Grids are persistent: 148 SMs x resident CTAs, grid-stride over tiles.
#include <cub/cub.cuh>

#include <atomic>
#include <climits>
#include <cstdlib>
#include <cstdio>

#include "kernels.cuh"

namespace psg {

namespace {
std::atomic<uint64_t> g_launches{0};
int g_sms = 0;
int sm_count() {
  if (g_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_sms <= 0) g_sms = 148;
  }
  return g_sms;
}
inline cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }
inline void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
inline unsigned grid_for(uint64_t n, int per_block) {
  uint64_t b = (n + per_block - 1) / per_block;
  const uint64_t cap = static_cast<uint64_t>(sm_count()) * 16;
  if (b > cap) b = cap;
  return static_cast<unsigned>(b < 1 ? 1 : b);
}

/// One 256-bit global store (sm_100: STG.256 - a whole 32-byte sector in one request).
__device__ __forceinline__ void st256(uint64_t* p, uint64_t a, uint64_t b, uint64_t c, uint64_t d) {
  asm volatile("st.global.v4.u64 [%0], {%1, %2, %3, %4};" ::"l"(p), "l"(a), "l"(b), "l"(c), "l"(d) : "memory");
}
}  // namespace

uint64_t kernel_launch_count() { return g_launches.load(); }
void count_external_launch() { count_launch(); }

// ------------------------------------------------------------------------------- fused k_scan
template <int R, int SINK>
__global__ void __launch_bounds__(kBlock) k_scan(const __grid_constant__ ScanProgram P, const Segment* __restrict__ segs,
                                                 const uint32_t* __restrict__ tile_seg, uint64_t ntiles) {
  extern __shared__ uint64_t smem[];  // [n_regs][R][kBlock]
  // Double-buffered tile descriptors: the next tile's segment/column pointers are fetched into
  // registers while the current tile computes (two dependent loads hidden behind the tile).
  __shared__ const uint64_t* s_col[2][kMaxIn];
  __shared__ uint64_t s_row0[2], s_rows[2];
  __shared__ uint32_t s_wcnt[R][kBlock / 32];
  __shared__ uint32_t s_woff[R][kBlock / 32];
  __shared__ unsigned long long s_base;
  __shared__ unsigned long long s_part[kMaxParts];
  __shared__ unsigned long long s_gacc[2 * kMaxSums + 1];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int TILE = R * kBlock;
#define V(reg, r) smem[((reg) * R + (r)) * kBlock + tid]

  if (SINK == SINK_MATERIALIZE && P.nparts > 1)
    for (int i = tid; i < P.nparts; i += kBlock) s_part[i] = 0;
  if (SINK == SINK_PROBE_GLOBAL || SINK == SINK_AGG_SCAN)
    for (int i = tid; i < 2 * kMaxSums + 1; i += kBlock) s_gacc[i] = 0;
  auto fetch = [&](uint64_t t, const uint64_t*& col, uint64_t& r0, uint64_t& rows) {
    const uint32_t si = __ldg(tile_seg + t);
    if (tid < P.n_in) {
      col = segs[si].col[tid];
    } else if (tid == kMaxIn) {
      const uint64_t tb = segs[si].tile_begin;
      r0 = (t - tb) * TILE;
      rows = min(static_cast<uint64_t>(TILE), segs[si].rows - r0);
    }
  };
  if (blockIdx.x < ntiles) {
    const uint64_t* c = nullptr;
    uint64_t r0 = 0, rows = 0;
    fetch(blockIdx.x, c, r0, rows);
    if (tid < P.n_in) s_col[0][tid] = c;
    if (tid == kMaxIn) s_row0[0] = r0, s_rows[0] = rows;
  }
  __syncthreads();

  int it = 0;
  for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const int b = it & 1;
    const uint64_t next = tile + gridDim.x;
    const uint64_t* pf_col = nullptr;
    uint64_t pf_r0 = 0, pf_rows = 0;
    if (next < ntiles) fetch(next, pf_col, pf_r0, pf_rows);
    const uint64_t* const* s_colb = s_col[b];
    const uint64_t row0 = s_row0[b];
    const int nrows = static_cast<int>(s_rows[b]);
#define s_col s_colb

    // Phase A: predicate columns for every row (R independent coalesced loads per column).
    uint32_t pass = 0;
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (r * kBlock + tid < nrows) pass |= 1u << r;
    for (int c = 0; c < P.n_pred; ++c) {
      const uint64_t* col = s_col[c] + row0;
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (pass & (1u << r)) V(c, r) = __ldcs(reinterpret_cast<const unsigned long long*>(col + r * kBlock + tid));
    }
    for (int a = 0; a < P.n_atoms; ++a) {
      const AtomDesc at = P.atoms[a];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (!(pass & (1u << r))) continue;
        const uint64_t v = V(at.reg, r);
        const bool ok = at.is_float ? cmp_f(__longlong_as_double(static_cast<long long>(v)), at.op,
                                            __longlong_as_double(static_cast<long long>(at.lit)))
                                    : cmp_i(static_cast<int64_t>(v), at.op, static_cast<int64_t>(at.lit));
        if (!ok) pass &= ~(1u << r);
      }
    }
    // Phase B: columns needed before joins / the sink key (late materialisation).
    for (int c = P.n_pred; c < P.n_early; ++c) {
      const uint64_t* col = s_col[c] + row0;
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (pass & (1u << r)) V(c, r) = __ldcs(reinterpret_cast<const unsigned long long*>(col + r * kBlock + tid));
    }
    // Phase C: unique-key local join chain (apply_chain, pipeline.cpp:431-448).
    for (int j = 0; j < P.n_joins; ++j) {
      const JoinDesc& jd = P.joins[j];
      uint64_t slot[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        slot[r] = ~0ULL;
        if (pass & (1u << r)) slot[r] = local_lookup(jd.t, V(jd.key_reg, r));
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (!(pass & (1u << r))) continue;
        if (slot[r] == ~0ULL) {
          pass &= ~(1u << r);
          continue;
        }
        const uint32_t st = jd.t.start[slot[r]];
        for (int p = 0; p < jd.t.npayload; ++p) V(jd.payload_reg[p], r) = jd.t.payload[p][st];
      }
    }

    if (SINK == SINK_PROBE || SINK == SINK_PROBE_GLOBAL) {
      const AggTableDev& t = P.agg;
      uint64_t slot[R];
      uint64_t home[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        slot[r] = ~0ULL;
        home[r] = 0;
        if (!(pass & (1u << r))) continue;
        const uint64_t key = V(P.key_reg, r);
        if (key == kEmptyKey) {
          slot[r] = (t.cold[(t.mask + 1) * t.cw] > 0) ? t.mask + 1 : ~0ULL;
          if (slot[r] == ~0ULL) pass &= ~(1u << r);
          continue;
        }
        if (!bloom_maybe(t, key)) {
          pass &= ~(1u << r);
          continue;
        }
        home[r] = slot_of(key, t.shift);
      }
      uint64_t k0[R];
#pragma unroll
      for (int r = 0; r < R; ++r)
        if ((pass & (1u << r)) && slot[r] == ~0ULL) k0[r] = t.hot[home[r] * t.hw];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (!(pass & (1u << r)) || slot[r] != ~0ULL) continue;
        slot[r] = agg_lookup_from(t, V(P.key_reg, r), home[r], k0[r]);
        if (slot[r] == ~0ULL) pass &= ~(1u << r);
      }
      // Late columns (sum inputs) only for matched rows.
      for (int c = P.n_early; c < P.n_in; ++c) {
        const uint64_t* col = s_col[c] + row0;
#pragma unroll
        for (int r = 0; r < R; ++r)
          if (pass & (1u << r)) V(c, r) = __ldcs(reinterpret_cast<const unsigned long long*>(col + r * kBlock + tid));
      }
      if (SINK == SINK_PROBE) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          if (!(pass & (1u << r))) continue;
          unsigned long long* h = reinterpret_cast<unsigned long long*>(t.hot + slot[r] * t.hw);
          atomicAdd(h + 1, 1ULL);
          for (int p = 0; p < P.n_sum; ++p) {
            const uint64_t v = V(P.sum_reg[p], r);
            if (t.ps_float[p])
              atomicAdd(reinterpret_cast<double*>(h + 2 + p), __longlong_as_double(static_cast<long long>(v)));
            else
              atomicAdd(h + 2 + p, static_cast<unsigned long long>(v));
          }
        }
      } else {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          if (!(pass & (1u << r))) continue;
          const uint64_t* cold = t.cold + slot[r] * t.cw;
          const uint64_t m = agg_mult(t, slot[r]);
          atomicAdd(&s_gacc[0], static_cast<unsigned long long>(m));
          for (int p = 0; p < P.n_sum; ++p) {
            const uint64_t v = V(P.sum_reg[p], r);
            if (t.ps_float[p])
              atomicAdd(reinterpret_cast<double*>(&s_gacc[1 + p]),
                        static_cast<double>(m) * __longlong_as_double(static_cast<long long>(v)));
            else
              atomicAdd(&s_gacc[1 + p], static_cast<unsigned long long>(m * v));
          }
          for (int b = 0; b < t.nbs; ++b) {
            if (t.bs_float[b])
              atomicAdd(reinterpret_cast<double*>(&s_gacc[1 + P.n_sum + b]),
                        __longlong_as_double(static_cast<long long>(cold[1 + b])));
            else
              atomicAdd(&s_gacc[1 + P.n_sum + b], static_cast<unsigned long long>(cold[1 + b]));
          }
        }
      }
    } else {
      // Remaining late columns for the other sinks.
      for (int c = P.n_early; c < P.n_in; ++c) {
        const uint64_t* col = s_col[c] + row0;
#pragma unroll
        for (int r = 0; r < R; ++r)
          if (pass & (1u << r)) V(c, r) = __ldcs(reinterpret_cast<const unsigned long long*>(col + r * kBlock + tid));
      }
      if (SINK == SINK_AGG_SCAN) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          if (!(pass & (1u << r))) continue;
          atomicAdd(&s_gacc[0], 1ULL);
          for (int p = 0; p < P.n_sum; ++p) {
            const uint64_t v = V(P.sum_reg[p], r);
            if (P.global_float[1 + p])
              atomicAdd(reinterpret_cast<double*>(&s_gacc[1 + p]), __longlong_as_double(static_cast<long long>(v)));
            else
              atomicAdd(&s_gacc[1 + p], static_cast<unsigned long long>(v));
          }
        }
      } else if (SINK == SINK_BUILD) {
        const AggTableDev& t = P.agg;
        // Claim the home slots of all R rows first (R CASes in flight), then resolve collisions.
        uint64_t slot[R];
        unsigned long long prev[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          slot[r] = ~0ULL;
          if (!(pass & (1u << r))) continue;
          const uint64_t key = V(P.key_reg, r);
          if (key == kEmptyKey) {
            slot[r] = t.mask + 1;
            prev[r] = kEmptyKey;
            continue;
          }
          slot[r] = slot_of(key, t.shift);
          prev[r] = atomicCAS(reinterpret_cast<unsigned long long*>(t.hot + slot[r] * t.hw), kEmptyKey, key);
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
          if (!(pass & (1u << r))) continue;
          const uint64_t key = V(P.key_reg, r);
          uint64_t s = slot[r];
          bool dup = prev[r] == key;
          if (prev[r] != kEmptyKey && prev[r] != key) s = agg_insert_from(t, key, (s + 1) & t.mask, dup);
          agg_count_build(t, key, s, dup);
          unsigned long long* cold = reinterpret_cast<unsigned long long*>(t.cold + s * t.cw);
          for (int b = 0; b < P.n_sum; ++b) {
            const uint64_t v = V(P.sum_reg[b], r);
            if (t.bs_float[b])
              atomicAdd(reinterpret_cast<double*>(cold + 1 + b), __longlong_as_double(static_cast<long long>(v)));
            else
              atomicAdd(cold + 1 + b, static_cast<unsigned long long>(v));
          }
        }
      } else {  // SINK_MATERIALIZE / SINK_COUNT
        if (SINK == SINK_MATERIALIZE && (P.semi_bloom != nullptr || P.semi_kbits != nullptr)) {
#pragma unroll
          for (int r = 0; r < R; ++r)
            if ((pass & (1u << r)) && !semi_maybe(P, V(P.semi_key_reg, r))) pass &= ~(1u << r);
        }
        uint32_t ballots[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          ballots[r] = __ballot_sync(0xffffffffu, (pass >> r) & 1u);
          if (lane == 0) s_wcnt[r][warp] = __popc(ballots[r]);
        }
        __syncthreads();
        if (tid == 0) {
          uint32_t acc = 0;
          for (int r = 0; r < R; ++r)
            for (int w = 0; w < kBlock / 32; ++w) {
              s_woff[r][w] = acc;
              acc += s_wcnt[r][w];
            }
          if (SINK == SINK_COUNT) {
            P.tile_counts[tile] = acc;
          } else if (P.tile_offsets != nullptr) {
            s_base = P.tile_offsets[tile];
          } else {
            s_base = acc ? atomicAdd(P.out_count, static_cast<unsigned long long>(acc)) : 0ULL;
          }
        }
        __syncthreads();
        if (SINK == SINK_MATERIALIZE) {
          const uint64_t base = s_base;
          const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
          for (int r = 0; r < R; ++r) {
            if (!((pass >> r) & 1u)) continue;
            const uint64_t pos = base + s_woff[r][warp] + __popc(ballots[r] & lt);
            if (pos >= P.out_cap) continue;  // host detects overflow via out_count
            for (int o = 0; o < P.n_out; ++o) P.out_col[o][pos] = V(P.out_reg[o], r);
            if (P.nparts > 1)
              atomicAdd(&s_part[part_of(V(P.part_key_reg, r), static_cast<uint32_t>(P.nparts))], 1ULL);
          }
        }
      }
    }
#undef s_col
    if (next < ntiles) {
      if (tid < P.n_in) s_col[b ^ 1][tid] = pf_col;
      if (tid == kMaxIn) s_row0[b ^ 1] = pf_r0, s_rows[b ^ 1] = pf_rows;
    }
    __syncthreads();
  }
#undef V
  if (SINK == SINK_MATERIALIZE && P.nparts > 1) {
    __syncthreads();
    for (int i = tid; i < P.nparts; i += kBlock)
      if (s_part[i]) atomicAdd(&P.part_counts[i], s_part[i]);
  }
  if (SINK == SINK_PROBE_GLOBAL || SINK == SINK_AGG_SCAN) {
    __syncthreads();
    const int n = 1 + P.n_sum + (SINK == SINK_PROBE_GLOBAL ? P.agg.nbs : 0);
    for (int i = tid; i < n; i += kBlock) {
      if (P.global_float[i])
        atomicAdd(reinterpret_cast<double*>(&P.global_acc[i]), __longlong_as_double(static_cast<long long>(s_gacc[i])));
      else
        atomicAdd(&P.global_acc[i], s_gacc[i]);
    }
  }
}

int scan_tile_rows() { return 4 * kBlock; }

template <int R, int SINK>
static void launch_scan_t(const ScanProgram& P, const Segment* d_segs, const uint32_t* d_tile_seg, uint64_t ntiles,
                          cudaStream_t st) {
  const size_t smem = static_cast<size_t>(P.n_regs < 1 ? 1 : P.n_regs) * R * kBlock * sizeof(uint64_t);
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(k_scan<R, SINK>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    configured = true;
  }
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_scan<R, SINK>, kBlock, smem);
  if (per_sm < 1) per_sm = 1;
  uint64_t grid = static_cast<uint64_t>(sm_count()) * per_sm;
  if (grid > ntiles) grid = ntiles;
  if (grid < 1) grid = 1;
  count_launch();
  k_scan<R, SINK><<<static_cast<unsigned>(grid), kBlock, smem, st>>>(P, d_segs, d_tile_seg, ntiles);
}

void launch_scan(const ScanProgram& P, const Segment* d_segs, const uint32_t* d_tile_seg, int nsegs, uint64_t ntiles,
                 void* stream) {
  if (ntiles == 0 || nsegs == 0) return;
  cudaStream_t st = S(stream);
  // Tiles are always 4 x 256 rows; programs with many registers use R=2 sub-tiles twice as
  // many CTAs would need, so they run R=4 with fewer resident CTAs (smem = n_regs * 8 KiB).
  switch (P.sink) {
    case SINK_MATERIALIZE: launch_scan_t<4, SINK_MATERIALIZE>(P, d_segs, d_tile_seg, ntiles, st); break;
    case SINK_BUILD: launch_scan_t<4, SINK_BUILD>(P, d_segs, d_tile_seg, ntiles, st); break;
    case SINK_PROBE: launch_scan_t<4, SINK_PROBE>(P, d_segs, d_tile_seg, ntiles, st); break;
    case SINK_PROBE_GLOBAL: launch_scan_t<4, SINK_PROBE_GLOBAL>(P, d_segs, d_tile_seg, ntiles, st); break;
    case SINK_COUNT: launch_scan_t<4, SINK_COUNT>(P, d_segs, d_tile_seg, ntiles, st); break;
    case SINK_AGG_SCAN: launch_scan_t<4, SINK_AGG_SCAN>(P, d_segs, d_tile_seg, ntiles, st); break;
  }
}

// ---------------------------------------------------------------------------- agg table setup
/// Hot slots initialised with 16-byte stores ({kEmptyKey, 0} then {0, 0}); cold is memset.
__global__ void k_agg_init(AggTableDev t, uint64_t nwords16) {
  ulonglong2* h = reinterpret_cast<ulonglong2*>(t.hot);
  const int per_slot = t.hw / 2;  // hw is even (2, 4, 8k)
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < nwords16;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    ulonglong2 v;
    v.x = (i % per_slot) == 0 ? kEmptyKey : 0ULL;
    v.y = 0ULL;
    h[i] = v;
  }
}
void launch_agg_init(const AggTableDev& t, uint64_t cap, void* stream) {
  count_launch();
  const uint64_t n16 = (cap + 1) * t.hw / 2;
  k_agg_init<<<grid_for(n16, 256), 256, 0, S(stream)>>>(t, n16);
  cudaMemsetAsync(t.cold, 0, (cap + 1) * t.cw * sizeof(uint64_t), S(stream));
  if (t.bloom) cudaMemsetAsync(t.bloom, 0, (t.bloom_mask + 1) * sizeof(uint32_t), S(stream));
}

__global__ void k_bloom_build(AggTableDev t, uint64_t cap) {
  for (uint64_t s = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; s < cap;
       s += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t key = t.hot[s * t.hw];
    if (key == kEmptyKey) continue;
    const uint64_t h2 = key * kBloomMul;
    atomicOr(t.bloom + (h2 >> t.bloom_shift), bloom_bits(h2, t.bloom_shift));
  }
}
void launch_bloom_build(const AggTableDev& t, uint64_t cap, void* stream) {
  if (!t.bloom) return;
  count_launch();
  k_bloom_build<<<grid_for(cap, 256), 256, 0, S(stream)>>>(t, cap);
}

// ------------------------------------------------------------------------------- local tables
__global__ void k_local_init(uint64_t* keys, uint32_t* cnt, uint64_t cap) {
  for (uint64_t s = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; s <= cap;
       s += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    if (s < cap) keys[s] = kEmptyKey;
    cnt[s] = 0;
  }
}
void launch_local_init(uint64_t* keys, uint32_t* cnt, uint64_t cap, void* stream) {
  count_launch();
  k_local_init<<<grid_for(cap + 1, 256), 256, 0, S(stream)>>>(keys, cnt, cap);
}

__global__ void k_local_count(uint64_t* keys, uint32_t* cnt, uint64_t mask, int shift, const uint64_t* bk, uint64_t n,
                              unsigned int* max_cnt) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t key = bk[i];
    uint64_t s;
    if (key == kEmptyKey) {
      s = mask + 1;
    } else {
      s = slot_of(key, shift);
      while (true) {
        const unsigned long long prev =
            atomicCAS(reinterpret_cast<unsigned long long*>(keys + s), kEmptyKey, key);
        if (prev == kEmptyKey || prev == key) break;
        s = (s + 1) & mask;
      }
    }
    const uint32_t old = atomicAdd(cnt + s, 1u);
    if (old > 0) atomicMax(max_cnt, old + 1);  // only duplicates contend
  }
}
void launch_local_count(uint64_t* keys, uint32_t* cnt, uint64_t mask, int shift, const uint64_t* bk, uint64_t n,
                        unsigned int* max_cnt, void* stream) {
  if (n == 0) return;
  count_launch();
  k_local_count<<<grid_for(n, 256), 256, 0, S(stream)>>>(keys, cnt, mask, shift, bk, n, max_cnt);
}

struct ColPtrs {
  const uint64_t* p[kMaxIn + kMaxPayload];
};
struct OutPtrs {
  uint64_t* p[kMaxIn + kMaxPayload];
};

__global__ void k_local_fill(const uint64_t* keys, const uint32_t* start, uint32_t* cursor, uint64_t mask, int shift,
                             const uint64_t* bk, ColPtrs src, OutPtrs dst, int ncols, uint64_t n) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t key = bk[i];
    uint64_t s;
    if (key == kEmptyKey) {
      s = mask + 1;
    } else {
      s = slot_of(key, shift);
      while (keys[s] != key) s = (s + 1) & mask;
    }
    const uint64_t pos = start[s] + atomicAdd(cursor + s, 1u);
    for (int c = 0; c < ncols; ++c) dst.p[c][pos] = src.p[c][i];
  }
}
void launch_local_fill(const uint64_t* keys, const uint32_t* start, uint32_t* cursor, uint64_t mask, int shift,
                       const uint64_t* bk, const uint64_t* const* src_cols, uint64_t* const* dst_cols, int ncols,
                       uint64_t n, void* stream) {
  if (n == 0) return;
  ColPtrs s{};
  OutPtrs d{};
  for (int c = 0; c < ncols; ++c) {
    s.p[c] = src_cols[c];
    d.p[c] = dst_cols[c];
  }
  count_launch();
  k_local_fill<<<grid_for(n, 256), 256, 0, S(stream)>>>(keys, start, cursor, mask, shift, bk, s, d, ncols, n);
}

size_t exclusive_scan_u32(const uint32_t* in, uint32_t* out, uint64_t n, void* tmp, size_t tmp_bytes, void* stream) {
  size_t bytes = tmp_bytes;
  cub::DeviceScan::ExclusiveSum(tmp, bytes, in, out, static_cast<int64_t>(n), S(stream));
  if (tmp) count_launch();
  return bytes;
}
size_t exclusive_scan_u64(const unsigned long long* in, unsigned long long* out, uint64_t n, void* tmp,
                          size_t tmp_bytes, void* stream) {
  size_t bytes = tmp_bytes;
  cub::DeviceScan::ExclusiveSum(tmp, bytes, in, out, static_cast<int64_t>(n), S(stream));
  if (tmp) count_launch();
  return bytes;
}

// --------------------------------------------------------------------- generic expanding join
__global__ void k_expand_count(LocalTableDev t, const uint64_t* pk, uint64_t n, uint32_t* counts) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t s = local_lookup(t, pk[i]);
    counts[i] = s == ~0ULL ? 0u : (t.bitmap ? 1u : t.cnt[s]);  // bitmap tables: unique keys, no payload
  }
}
void launch_expand_count(LocalTableDev t, const uint64_t* pk, uint64_t n, uint32_t* counts, void* stream) {
  if (n == 0) return;
  count_launch();
  k_expand_count<<<grid_for(n, 256), 256, 0, S(stream)>>>(t, pk, n, counts);
}

__global__ void k_expand_write(LocalTableDev t, const uint64_t* pk, uint64_t n, const uint32_t* off, ColPtrs probe,
                               int nprobe, OutPtrs out) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t s = local_lookup(t, pk[i]);
    if (s == ~0ULL) continue;
    const uint32_t c = t.bitmap ? 1u : t.cnt[s], st = t.bitmap ? 0u : t.start[s];
    const uint64_t o = off[i];
    for (uint32_t k = 0; k < c; ++k) {
      for (int p = 0; p < t.npayload; ++p) out.p[p][o + k] = t.payload[p][st + k];
      for (int q = 0; q < nprobe; ++q) out.p[t.npayload + q][o + k] = probe.p[q][i];
    }
  }
}
void launch_expand_write(LocalTableDev t, const uint64_t* pk, uint64_t n, const uint32_t* offsets,
                         const uint64_t* const* probe_cols, int nprobe, uint64_t* const* out_cols, void* stream) {
  if (n == 0) return;
  ColPtrs pc{};
  OutPtrs oc{};
  for (int q = 0; q < nprobe; ++q) pc.p[q] = probe_cols[q];
  for (int c = 0; c < t.npayload + nprobe; ++c) oc.p[c] = out_cols[c];
  count_launch();
  k_expand_write<<<grid_for(n, 256), 256, 0, S(stream)>>>(t, pk, n, offsets, pc, nprobe, oc);
}

// ------------------------------------------------------------------------ partition / scatter
/// Scatter into dest-major send slabs. Each block takes 4096-row chunks: positions inside the chunk
/// come from warp-aggregated shared-memory counters (one shared atomic per (warp, dest)), then one
/// global atomic per (block, dest) reserves the chunk's range in each destination's slab.
constexpr int kScatterPer = 16;  // rows per thread per chunk
__global__ void __launch_bounds__(256) k_part_scatter(ColPtrs in, int ncols, uint64_t n, int key_col, int nparts,
                                                      const unsigned long long* dest_base,
                                                      const unsigned long long* dest_cnt, unsigned long long* cursor,
                                                      uint64_t* send, KeyField kf) {
  __shared__ unsigned int s_cnt[kMaxParts];
  __shared__ unsigned long long s_base[kMaxParts];
  const int tid = threadIdx.x, lane = tid & 31;
  for (int d = tid; d < nparts; d += 256) s_cnt[d] = 0;
  __syncthreads();
  constexpr uint64_t kChunk = 256ULL * kScatterPer;
  for (uint64_t c0 = blockIdx.x * kChunk; c0 < n; c0 += static_cast<uint64_t>(gridDim.x) * kChunk) {
    uint32_t dest[kScatterPer], pos[kScatterPer];
#pragma unroll
    for (int k = 0; k < kScatterPer; ++k) {
      const uint64_t i = c0 + k * 256 + tid;
      const bool valid = i < n;
      uint64_t key = valid ? in.p[key_col][i] : 0;
      if (kf.mask) key = static_cast<uint64_t>(kf.min) + ((key >> kf.shift) & kf.mask);  // bit-packed rows
      const uint32_t d = valid ? part_of(key, static_cast<uint32_t>(nparts)) : 0xffffffffu;
      const unsigned peers = __match_any_sync(0xffffffffu, d);
      const int leader = __ffs(peers) - 1;
      unsigned int old = 0;
      if (valid && lane == leader) old = atomicAdd(&s_cnt[d], static_cast<unsigned int>(__popc(peers)));
      old = __shfl_sync(0xffffffffu, old, leader);
      dest[k] = d;
      pos[k] = old + __popc(peers & ((1u << lane) - 1u));
    }
    __syncthreads();
    for (int d = tid; d < nparts; d += 256) {
      s_base[d] = s_cnt[d] ? atomicAdd(cursor + d, static_cast<unsigned long long>(s_cnt[d])) : 0ULL;
      s_cnt[d] = 0;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kScatterPer; ++k) {
      const uint64_t i = c0 + k * 256 + tid;
      if (i >= n) continue;
      const uint32_t d = dest[k];
      const uint64_t at = s_base[d] + pos[k];
      const uint64_t cnt = dest_cnt[d];
      uint64_t* region = send + dest_base[d] * static_cast<uint64_t>(ncols);
      for (int c = 0; c < ncols; ++c) region[c * cnt + at] = in.p[c][i];
    }
  }
}
void launch_part_scatter(const uint64_t* const* in_cols, int ncols, uint64_t n, int key_col, int nparts,
                         const unsigned long long* dest_base, const unsigned long long* dest_cnt,
                         unsigned long long* cursor, uint64_t* send, void* stream, KeyField kf) {
  if (n == 0) return;
  ColPtrs pc{};
  for (int c = 0; c < ncols; ++c) pc.p[c] = in_cols[c];
  count_launch();
  uint64_t blocks = (n + 256ULL * kScatterPer - 1) / (256ULL * kScatterPer);
  const uint64_t maxb = static_cast<uint64_t>(sm_count()) * 8;
  if (blocks > maxb) blocks = maxb;
  k_part_scatter<<<static_cast<unsigned>(blocks), 256, 0, S(stream)>>>(pc, ncols, n, key_col, nparts, dest_base, dest_cnt,
                                                                      cursor, send, kf);
}

__global__ void k_part_ids(const uint64_t* keys, uint64_t n, int nparts, int identity, uint32_t* ids) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t k = keys[i];
    ids[i] = identity ? static_cast<uint32_t>(k % static_cast<uint64_t>(nparts)) : part_of(k, nparts);
  }
}
void launch_part_ids(const uint64_t* keys, uint64_t n, int nparts, int identity, uint32_t* ids, void* stream) {
  if (n == 0) return;
  count_launch();
  k_part_ids<<<grid_for(n, 256), 256, 0, S(stream)>>>(keys, n, nparts, identity, ids);
}

__global__ void k_gather(ColPtrs in, int ncols, const uint32_t* idx, uint64_t n, OutPtrs out) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t j = idx[i];
    for (int c = 0; c < ncols; ++c) out.p[c][i] = in.p[c][j];
  }
}
void launch_gather(const uint64_t* const* in_cols, int ncols, const uint32_t* idx, uint64_t n, uint64_t* const* out,
                   void* stream) {
  if (n == 0) return;
  ColPtrs pc{};
  OutPtrs oc{};
  for (int c = 0; c < ncols; ++c) {
    pc.p[c] = in_cols[c];
    oc.p[c] = out[c];
  }
  count_launch();
  k_gather<<<grid_for(n, 256), 256, 0, S(stream)>>>(pc, ncols, idx, n, oc);
}

/// out[c][i] = in[c][idx[i]] with 64-bit indices (row indices produced by an expanding join).
__global__ void k_gather64(ColPtrs in, int ncols, const uint64_t* idx, uint64_t n, OutPtrs out) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t j = idx[i];
    for (int c = 0; c < ncols; ++c) out.p[c][i] = in.p[c][j];
  }
}
void launch_gather64(const uint64_t* const* in_cols, int ncols, const uint64_t* idx, uint64_t n, uint64_t* const* out,
                     void* stream) {
  if (n == 0 || ncols == 0) return;
  ColPtrs pc{};
  OutPtrs oc{};
  for (int c = 0; c < ncols; ++c) {
    pc.p[c] = in_cols[c];
    oc.p[c] = out[c];
  }
  count_launch();
  k_gather64<<<grid_for(n, 256), 256, 0, S(stream)>>>(pc, ncols, idx, n, oc);
}

/// Interleaved rank records: krec[2w] = 64-bit bitmap word w, krec[2w+1] = krank[w] (one 16-byte
/// load per probe instead of two 4/8-byte loads from two arrays).
__global__ void k_krec_build(const unsigned long long* __restrict__ bits, const uint32_t* __restrict__ krank, uint64_t n,
                             unsigned long long* __restrict__ krec) {
  for (uint64_t w = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; w < n;
       w += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    ulonglong2 v;
    v.x = bits[w];
    v.y = krank[w];
    reinterpret_cast<ulonglong2*>(krec)[w] = v;
  }
}
constexpr int kRankThreads = 256, kRankIters = 8;
constexpr uint64_t kRankTile = kRankThreads * kRankIters;  // words per CTA
uint64_t rank_tiles(uint64_t n) { return (n + kRankTile - 1) / kRankTile; }
__global__ void __launch_bounds__(kRankThreads) k_rank_tiles(const unsigned long long* __restrict__ bits, uint64_t n,
                                                             uint32_t* __restrict__ tile_sums) {
  const uint64_t base = blockIdx.x * kRankTile;
  uint32_t c = 0;
#pragma unroll
  for (int it = 0; it < kRankIters; ++it) {
    const uint64_t w = base + it * kRankThreads + threadIdx.x;
    if (w < n) c += __popcll(bits[w]);
  }
  c = __reduce_add_sync(0xffffffffu, c);
  __shared__ uint32_t ws[kRankThreads / 32];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x < 32) {
    uint32_t v = threadIdx.x < kRankThreads / 32 ? ws[threadIdx.x] : 0;
    v = __reduce_add_sync(0xffffffffu, v);
    if (threadIdx.x == 0) tile_sums[blockIdx.x] = v;
  }
}
__global__ void __launch_bounds__(kRankThreads) k_rank_build(const unsigned long long* __restrict__ bits, uint64_t n,
                                                             const uint32_t* __restrict__ tile_sums,
                                                             uint32_t* __restrict__ krank,
                                                             unsigned long long* __restrict__ krec) {
  __shared__ uint32_t ws[kRankThreads / 32];
  __shared__ uint32_t s_run;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  // this tile's offset: the sum of the earlier tiles' counts (<= a few thousand words, from L2)
  uint32_t pre = 0;
  for (uint32_t t = threadIdx.x; t < blockIdx.x; t += kRankThreads) pre += tile_sums[t];
  pre = __reduce_add_sync(0xffffffffu, pre);
  if (lane == 0) ws[wid] = pre;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t v = 0;
    for (int k = 0; k < kRankThreads / 32; ++k) v += ws[k];
    s_run = v;
  }
  __syncthreads();
  const uint64_t base = blockIdx.x * kRankTile;
  for (int it = 0; it < kRankIters; ++it) {
    const uint64_t w = base + it * kRankThreads + threadIdx.x;
    const unsigned long long b = w < n ? bits[w] : 0ULL;
    const uint32_t c = __popcll(b);
    uint32_t inc = c;  // inclusive warp scan
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, inc, d);
      if (lane >= d) inc += y;
    }
    if (lane == 31) ws[wid] = inc;
    __syncthreads();
    uint32_t wpre = 0;
    for (int k = 0; k < wid; ++k) wpre += ws[k];
    const uint32_t r = s_run + wpre + inc - c;
    if (w < n) {
      krank[w] = r;
      ulonglong2 v;
      v.x = b;
      v.y = r;
      reinterpret_cast<ulonglong2*>(krec)[w] = v;
    }
    __syncthreads();  // every warp has read ws and s_run
    if (threadIdx.x == kRankThreads - 1) s_run = r + c;
    __syncthreads();
  }
}
void launch_rank_records(const unsigned long long* bits, uint64_t n, uint32_t* tile_sums, uint32_t* krank,
                         unsigned long long* krec, void* stream) {
  if (n == 0) return;
  const uint64_t tiles = rank_tiles(n);
  count_launch();
  k_rank_tiles<<<static_cast<unsigned>(tiles), kRankThreads, 0, S(stream)>>>(bits, n, tile_sums);
  count_launch();
  k_rank_build<<<static_cast<unsigned>(tiles), kRankThreads, 0, S(stream)>>>(bits, n, tile_sums, krank, krec);
}
void launch_krec_build(const unsigned long long* bits, const uint32_t* krank, uint64_t n, unsigned long long* krec,
                       void* stream) {
  if (n == 0) return;
  count_launch();
  k_krec_build<<<grid_for(n, 256), 256, 0, S(stream)>>>(bits, krank, n, krec);
}

/// Owner bitmap at N > 1: own[w] = the bits of the global key bitmap word w whose key this rank
/// owns (partition_of(key) == self). cnt[0] += own bits, cnt[1] += global bits (the engine checks
/// the global count against the rows that set it: a SUM all-reduce of overlapping bitmaps carries).
__global__ void k_own_mask(const unsigned long long* __restrict__ global, unsigned long long* __restrict__ own,
                           uint64_t nwords, int64_t kmin, int nparts, int self, unsigned long long* cnt) {
  unsigned long long no = 0, ng = 0;
  for (uint64_t w = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; w < nwords;
       w += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    unsigned long long g = global[w], m = 0, rest = g;
    const uint64_t base = static_cast<uint64_t>(kmin) + (w << 6);
    while (rest) {
      const int b = __ffsll(static_cast<long long>(rest)) - 1;
      rest &= rest - 1;
      if (part_of(base + b, static_cast<uint32_t>(nparts)) == static_cast<uint32_t>(self)) m |= 1ULL << b;
    }
    own[w] = m;
    no += __popcll(m);
    ng += __popcll(g);
  }
  no = __reduce_add_sync(0xffffffffu, static_cast<unsigned>(no));
  ng = __reduce_add_sync(0xffffffffu, static_cast<unsigned>(ng));
  if ((threadIdx.x & 31) == 0 && (no | ng)) {
    atomicAdd(cnt, no);
    atomicAdd(cnt + 1, ng);
  }
}
void launch_own_mask(const unsigned long long* global, unsigned long long* own, uint64_t nwords, int64_t kmin, int nparts,
                     int self, unsigned long long* cnt, void* stream) {
  if (nwords == 0) return;
  count_launch();
  k_own_mask<<<grid_for(nwords, 256), 256, 0, S(stream)>>>(global, own, nwords, kmin, nparts, self, cnt);
}

/// Global key bitmap at N > 1 without a collective: every rank's local bitmap (set by its build
/// scan) lives in the symmetric heap, and each rank ORs all of them word by word through NVLink
/// (16-byte loads), keeping the owned bits too. Keys two ranks both hold (duplicates: the rank
/// table needs unique keys) show as a word whose summed popcounts exceed the popcount of the OR
/// (cnt[2]); a key repeated within a rank, or outside the range, as fewer global bits than the
/// summed row counts of the ranks' build scans (cnt[3], read from their heaps). Identical on every
/// rank (same inputs): the re-run decision needs no all-reduce. cnt[0] += own bits, cnt[1] +=
/// global bits.
uint32_t own_period(int nparts) {
  if (nparts < 2 || (nparts & (nparts - 1)) != 0 || nparts > kMaxSlabPeers) return 0;
  return 128u * static_cast<uint32_t>(nparts);  // 2^(13 + log2 n) keys / 64 per word
}
__global__ void k_own_table(int64_t kmin, int nparts, int self, uint32_t period, unsigned long long* table) {
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= period) return;
  const uint64_t base = static_cast<uint64_t>(kmin) + (static_cast<uint64_t>(j) << 6);
  unsigned long long m = 0;
  for (int b = 0; b < 64; ++b)
    if (part_of(base + b, static_cast<uint32_t>(nparts)) == static_cast<uint32_t>(self)) m |= 1ULL << b;
  table[j] = m;
}
void launch_own_table(int64_t kmin, int nparts, int self, unsigned long long* table, void* stream) {
  const uint32_t period = own_period(nparts);
  if (!period) return;
  count_launch();
  k_own_table<<<(period + 127) / 128, 128, 0, S(stream)>>>(kmin, nparts, self, period, table);
}

__global__ void k_or_own(OrPeers p, uint64_t nwords, int64_t kmin, int self, unsigned long long* __restrict__ global,
                         unsigned long long* __restrict__ own, unsigned long long* cnt,
                         const unsigned long long* __restrict__ table, uint32_t period) {
  unsigned long long no = 0, ng = 0;
  bool dup = false;
  if (blockIdx.x == 0 && threadIdx.x < p.n)  // every rank's row count: sum == global bits unless keys repeat
    atomicAdd(cnt + 3, *reinterpret_cast<const volatile unsigned long long*>(p.rows[threadIdx.x]));
  const uint64_t npairs = nwords / 2;
  auto word = [&](uint64_t w, unsigned long long g, int s) {
    if (s != __popcll(g)) dup = true;
    unsigned long long m = 0, rest = g;
    if (table) {
      m = g & __ldg(table + (w & (period - 1)));
      rest = 0;
    }
    const uint64_t base = static_cast<uint64_t>(kmin) + (w << 6);
    while (rest) {
      const int b = __ffsll(static_cast<long long>(rest)) - 1;
      rest &= rest - 1;
      if (part_of(base + b, static_cast<uint32_t>(p.n)) == static_cast<uint32_t>(self)) m |= 1ULL << b;
    }
    global[w] = g;
    own[w] = m;
    no += __popcll(m);
    ng += __popcll(g);
  };
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < npairs;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    unsigned long long g0 = 0, g1 = 0;
    int s0 = 0, s1 = 0;
    for (int r = 0; r < p.n; ++r) {
      const ulonglong2 x = __ldcs(reinterpret_cast<const ulonglong2*>(p.bits[r]) + i);
      g0 |= x.x, g1 |= x.y;
      s0 += __popcll(x.x), s1 += __popcll(x.y);
    }
    word(2 * i, g0, s0);
    word(2 * i + 1, g1, s1);
  }
  if ((nwords & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long g = 0;
    int sc = 0;
    for (int r = 0; r < p.n; ++r) {
      const unsigned long long x = p.bits[r][nwords - 1];
      g |= x;
      sc += __popcll(x);
    }
    word(nwords - 1, g, sc);
  }
  no = __reduce_add_sync(0xffffffffu, static_cast<unsigned>(no));
  ng = __reduce_add_sync(0xffffffffu, static_cast<unsigned>(ng));
  const unsigned anydup = __ballot_sync(0xffffffffu, dup);
  if ((threadIdx.x & 31) == 0) {
    if (no | ng) {
      atomicAdd(cnt, no);
      atomicAdd(cnt + 1, ng);
    }
    if (anydup) atomicOr(cnt + 2, 1ULL);
  }
}
void launch_or_own(const OrPeers& p, uint64_t nwords, int64_t kmin, int self, unsigned long long* global,
                   unsigned long long* own, unsigned long long* cnt, void* stream, const unsigned long long* own_table,
                   uint32_t own_period) {
  if (nwords == 0) return;
  count_launch();
  int sms = 148, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  k_or_own<<<sms * 8, 256, 0, S(stream)>>>(p, nwords, kmin, self, global, own, cnt, own_table,
                                           own_table ? own_period : 0);
}

__global__ void k_peer_barrier(PeerFlags f, const uint32_t* own, int self, int n, uint32_t epoch, unsigned int* err) {
  const int i = threadIdx.x;
  if (i >= n) return;
  __threadfence_system();
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(f.flag[i] + self), "r"(epoch) : "memory");
  const long long t0 = clock64();
  while (true) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(own + i) : "memory");
    if (static_cast<int32_t>(v - epoch) >= 0) break;
    if (clock64() - t0 > (20LL << 30)) {  // ~10 s at 2 GHz: a rank never arrived
      atomicExch(err, 1u);
      break;
    }
    __nanosleep(32);
  }
}
void launch_peer_barrier(const PeerFlags& f, const uint32_t* own, int self, int n, uint32_t epoch, unsigned int* err,
                         void* stream) {
  count_launch();
  k_peer_barrier<<<1, 32, 0, S(stream)>>>(f, own, self, n, epoch, err);
}

__global__ void k_gather_words(GatherWords g, unsigned long long* host) {
  const int i = threadIdx.x;
  if (i < g.n)
    host[i] = (g.w32 >> i) & 1 ? static_cast<unsigned long long>(*static_cast<const uint32_t*>(g.src[i]))
                               : *static_cast<const unsigned long long*>(g.src[i]);
  __threadfence_system();
}
void launch_gather_words(const GatherWords& g, unsigned long long* host_mapped, void* stream) {
  if (g.n <= 0) return;
  count_launch();
  k_gather_words<<<1, 32, 0, S(stream)>>>(g, host_mapped);
}

/// L2 warm-up of a table the next kernel reads at random (the owner-side fold's rank records: the
/// probe kernel touched only the records of the rows this rank owned, so the received rows' records
/// are cold and each fold lookup went to DRAM): bulk L2 prefetches of 64 KB per instruction, issued
/// before the cross-rank barrier so they overlap the wait.
__global__ void k_l2_prefetch(const unsigned char* p, uint64_t bytes) {
  constexpr uint64_t kChunk = 64ull << 10;
  for (uint64_t off = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) * kChunk; off < bytes;
       off += static_cast<uint64_t>(gridDim.x) * blockDim.x * kChunk) {
    const uint32_t n = static_cast<uint32_t>(min(kChunk, bytes - off)) & ~15u;
    if (n) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p + off), "r"(n) : "memory");
  }
}
/// The same warm-up by loads that mark the lines evict-last (one 16-byte load per 128-byte line).
__global__ void k_l2_touch(const unsigned long long* p, uint64_t lines, unsigned long long* sink) {
  const uint64_t pol = l2_evict_last();
  unsigned long long acc = 0;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < lines;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    uint64_t a, b;
    ldg_keep_v2u64(p + 16 * i, pol, a, b);
    acc ^= a ^ b;
  }
  if (acc == 0x9E3779B97F4A7C15ULL) *sink = acc;  // (keeps the loads)
}
void launch_l2_prefetch(const void* p, uint64_t bytes, void* stream) {
  if (!p || bytes < 16) return;
  count_launch();
  static const int mode = [] {
    const char* e = std::getenv("PSG_CONSUME_PREFETCH");
    return e ? std::atoi(e) : 0;
  }();
  if (mode == 2) {
    static unsigned long long* sink = nullptr;
    if (!sink) cudaMalloc(&sink, 8);
    k_l2_touch<<<sm_count() * 8, 256, 0, S(stream)>>>(static_cast<const unsigned long long*>(p), bytes / 128, sink);
  } else {
    k_l2_prefetch<<<64, 32, 0, S(stream)>>>(static_cast<const unsigned char*>(p), bytes);
  }
}

/// Peer-slab shuffle, owner side: every packed row the other ranks stored into this rank's
/// receive slab (region r = source r, *c.src_cnt[r] rows, read from the source's counters through
/// NVLink after the cross-rank barrier) is unpacked, finds its slot in the rank-indexed table
/// (one 16-byte rank record) and is appended to the slot's aggregation bucket - the same entry
/// the probe kernel appends for the rows it owns (ScanProgram::bkt).
__global__ void __launch_bounds__(256) k_slab_consume(AggTableDev t, SlabConsume c) {
  const uint64_t gtid = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  __shared__ unsigned long long s_n[kMaxSlabPeers];  // one NVLink read per (block, source)
  if (threadIdx.x < c.nsrc)
    s_n[threadIdx.x] = c.src_cnt[threadIdx.x] == nullptr
                           ? 0ULL
                           : *reinterpret_cast<const volatile unsigned long long*>(c.src_cnt[threadIdx.x]);
  __syncthreads();
  for (int src = 0; src < c.nsrc; ++src) {
    const uint64_t n = min(static_cast<uint64_t>(s_n[src]), c.cap);
    if (n == 0) continue;
    if (gtid == 0) atomicAdd(c.received, static_cast<unsigned long long>(n));
    const uint64_t* in = c.src_rows[src];
    // 4 rows per thread per round: their loads (NVLink in the pull mode) and rank-record lookups
    // are in flight together before the dependent appends
    constexpr int U = 4;
    for (uint64_t i0 = gtid; i0 < n; i0 += U * stride) {
      uint64_t w[U], d[U];
      ulonglong2 rec[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint64_t i = i0 + u * stride;
        w[u] = i < n ? __ldcs(reinterpret_cast<const unsigned long long*>(in + i)) : 0ULL;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint64_t key = static_cast<uint64_t>(c.pmin[0]) + ((w[u] >> c.pshift[0]) & c.pmask[0]);
        d[u] = i0 + u * stride < n && !(w[u] >> 63) ? key - static_cast<uint64_t>(t.kmin) : ~0ULL;
        rec[u] = d[u] < t.krange ? __ldg(reinterpret_cast<const ulonglong2*>(t.krec) + (d[u] >> 6)) : make_ulonglong2(0, 0);
      }
      // the U reservations in flight together, then the stores (one atomic round trip per round)
      uint64_t slot[U], e[U], bk[U];
      unsigned pos[U];
      bool ok[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        // (padding of partly filled chunks: bit 63; the senders' global screen guarantees membership)
        ok[u] = d[u] < t.krange && ((rec[u].x >> (d[u] & 63)) & 1ULL);
        slot[u] = ok[u] ? rec[u].y + static_cast<uint64_t>(__popcll(rec[u].x & ((1ULL << (d[u] & 63)) - 1ULL))) : 0;
        e[u] = slot[u] & static_cast<uint64_t>(kBucketSlots - 1);
        for (int k = 0; k + 1 < c.npack; ++k) {
          const uint64_t v = static_cast<uint64_t>(c.pmin[1 + k]) + ((w[u] >> c.pshift[1 + k]) & c.pmask[1 + k]);
          e[u] |= ((v - static_cast<uint64_t>(c.bmin[k])) & c.bmask[k]) << c.bshift[k];
        }
        bk[u] = ((slot[u] >> kBucketBits) << c.bsub_bits) | (threadIdx.x & ((1u << c.bsub_bits) - 1u));
        pos[u] = 0;
        if (ok[u] && !(c.diag & 4)) pos[u] = atomicAdd(c.fill + bk[u], 1u);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (!ok[u]) continue;
        if (c.diag & 4) {  // measurement only (PSG_SLAB_DIAG=4): no bucket append
          if (e[u] == ~0ULL) c.bkt[bk[u]] = e[u];
          continue;
        }
        if (pos[u] < c.bcap) {
          c.bkt[bk[u] * c.bcap + pos[u]] = e[u];
        } else {
          const unsigned o = atomicAdd(c.ovf_count, 1u);
          if (o < c.ovf_cap) {
            c.ovf[2 * o] = slot[u];
            c.ovf[2 * o + 1] = e[u];
          }
        }
      }
    }
  }
}
void launch_slab_consume(const AggTableDev& t, const SlabConsume& c, void* stream) {
  count_launch();
  int sms = 148, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // PSG_CONSUME_BPS: blocks per SM (measurement knob)
  static const int bps = [] {
    const char* e = std::getenv("PSG_CONSUME_BPS");
    return e ? std::max(1, std::atoi(e)) : 4;
  }();
  k_slab_consume<<<sms * bps, 256, 0, S(stream)>>>(t, c);
}

/// Output column recipe of the emit kernels: kind 0 key, 1 rows, 2 probe sum idx, 3 build sum idx.
struct EmitCols {
  int32_t kind[2 * kMaxSums + 2];
  int32_t idx[2 * kMaxSums + 2];
};

/// Bucketed aggregation, finalisation (one CTA per bucket of kBucketSlots consecutive rank-table
/// slots; ScanProgram::bkt). The probe appended one word per surviving row to its slot's bucket
/// (slot low bits + offset-encoded probe sums); entries past the bucket capacity were added
/// straight into the (zeroed) hot table instead. Pass 1 counts the groups (slots with hits) per
/// bucket, an exclusive scan turns the counts into output offsets, and pass 2 folds the bucket in
/// shared memory and writes its result rows in key order: keys come from the key bitmap (slot =
/// krank[w] + set bits below), so the table in HBM is never read or written on the common path.
namespace {
__device__ __forceinline__ uint64_t bucket_value(const BucketDev& b, uint64_t w, int k) {
  return static_cast<uint64_t>(b.min[k]) + ((w >> b.shift[k]) & b.mask[k]);
}
}  // namespace

/// First key-bitmap word of every bucket: word w holds slots [krank[w], krank[w+1]), so bucket b
/// (first slot b * kBucketSlots) starts in the w whose range contains it.
__global__ void k_bucket_words(AggTableDev t, uint64_t nwords, uint64_t nslots, uint32_t* first_word) {
  for (uint64_t w = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; w < nwords;
       w += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t lo = t.krank[w], hi = w + 1 < nwords ? t.krank[w + 1] : nslots;
    for (uint64_t b = (lo + kBucketSlots - 1) >> kBucketBits; (b << kBucketBits) < hi; ++b)
      first_word[b] = static_cast<uint32_t>(w);
  }
}

/// Shared-memory fold of one bucket: hits[i] (u32) and, per probe sum k, the 64-bit sum of the
/// offset-encoded fields as two u32 words (lo with carry into hi: native 32-bit shared atomics; a
/// 64-bit shared atomicAdd compiles to a CAS loop). sum_k = fields + hits * bkt_min[k] (mod 2^64).
struct BucketSmem {
  uint32_t* hits;
  uint32_t* lo;  // [nps][kBucketSlots]
  uint32_t* hi;
  uint16_t* pos;
};
__device__ __forceinline__ BucketSmem bucket_smem(unsigned char* base, int nps) {
  BucketSmem m;
  m.hits = reinterpret_cast<uint32_t*>(base);
  m.lo = m.hits + kBucketSlots;
  m.hi = m.lo + nps * kBucketSlots;
  m.pos = reinterpret_cast<uint16_t*>(m.hi + nps * kBucketSlots);
  return m;
}
__device__ __forceinline__ void add64_u32pair(uint32_t* lo, uint32_t* hi, uint64_t v) {
  const uint32_t vl = static_cast<uint32_t>(v), vh = static_cast<uint32_t>(v >> 32);
  const uint32_t old = atomicAdd(lo, vl);
  const uint32_t carry = (old + vl) < old ? 1u : 0u;
  if (vh + carry) atomicAdd(hi, vh + carry);
}

/// Single pass with decoupled look-back: a CTA claims the next bucket from a ticket (so every
/// lower bucket is already owned by a running CTA), folds it, publishes its group count, adds up
/// its predecessors' published counts/prefixes for its output offset, publishes its inclusive
/// prefix and writes its rows. state[b] = (status << 62) | value: 1 = count, 2 = inclusive prefix.
__global__ void __launch_bounds__(512) k_bucket_emit(AggTableDev t, BucketDev b, uint64_t nslots, uint64_t nwords,
                                                     unsigned long long* state, unsigned int* ticket,
                                                     const uint32_t* first_word, int nc, EmitCols ec, uint64_t* out,
                                                     uint64_t nbuckets) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int nps = t.nps;
  const BucketSmem m = bucket_smem(smem_raw, nps);
  __shared__ uint32_t s_warp[16];
  __shared__ uint64_t s_bucket, s_base;
  // persistent CTAs (at most the resident count, so every claimed predecessor is running): each
  // claims buckets from the ticket in order until none is left
  for (;;) {
  if (threadIdx.x == 0) s_bucket = atomicAdd(ticket, 1u);
  for (int i = threadIdx.x; i < (1 + 2 * nps) * kBucketSlots; i += blockDim.x) m.hits[i] = 0;
  __syncthreads();
  if (s_bucket >= nbuckets) return;
  const uint64_t bucket = s_bucket, s0 = bucket << kBucketBits;
  const uint64_t s_end = min(s0 + kBucketSlots, nslots);
  for (uint64_t sub = bucket << b.sub_bits; sub < (bucket + 1) << b.sub_bits; ++sub) {
    const uint32_t n = min(b.fill[sub], b.cap);
    const uint64_t* e = b.bkt + sub * b.cap;
    // 4 entries per thread per round: their loads are in flight together before the folds
    for (uint32_t i0 = threadIdx.x; i0 < n; i0 += 4 * blockDim.x) {
      uint64_t w4[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t i = i0 + u * blockDim.x;
        w4[u] = i < n ? __ldcs(reinterpret_cast<const unsigned long long*>(e + i)) : 0ULL;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (i0 + u * blockDim.x >= n) break;
        const uint64_t w = w4[u];
        const uint32_t sl = static_cast<uint32_t>(w & (kBucketSlots - 1));
        atomicAdd(&m.hits[sl], 1u);
        for (int k = 0; k < nps; ++k)
          add64_u32pair(&m.lo[k * kBucketSlots + sl], &m.hi[k * kBucketSlots + sl], (w >> b.shift[k]) & b.mask[k]);
      }
    }
  }
  __syncthreads();
  // rows that found a bucket full sit in the overflow list (rare; empty on the common path)
  const uint32_t novf = min(*b.ovf_count, b.ovf_cap);
  for (uint32_t i = threadIdx.x; i < novf; i += blockDim.x) {
    const uint64_t slot = b.ovf[2 * i];
    if ((slot >> kBucketBits) != bucket) continue;
    const uint64_t w = b.ovf[2 * i + 1];
    const uint32_t sl = static_cast<uint32_t>(slot & (kBucketSlots - 1));
    atomicAdd(&m.hits[sl], 1u);
    for (int k = 0; k < nps; ++k) add64_u32pair(&m.lo[k * kBucketSlots + sl], &m.hi[k * kBucketSlots + sl], (w >> b.shift[k]) & b.mask[k]);
  }
  __syncthreads();
  // exclusive prefix of "slot has hits" over the bucket: warp w owns slots [w * per32 * 32, ...) as
  // per32 rows of 32 consecutive slots, lane = slot within the row (conflict-free shared reads);
  // ballots give the in-row prefix, row totals the in-warp prefix, warp totals the rest
  constexpr int per32 = kBucketSlots / 512;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int wbase = wid * per32 * 32;
  uint32_t wsum = 0;
  unsigned flags[per32];
#pragma unroll
  for (int k = 0; k < per32; ++k) {
    const int i = wbase + k * 32 + lane;
    flags[k] = __ballot_sync(0xffffffffu, m.hits[i] != 0 && s0 + i < s_end);
    wsum += __popc(flags[k]);
  }
  if (lane == 0) s_warp[wid] = wsum;
  __syncthreads();
  uint32_t acc = 0;
  for (int w = 0; w < wid; ++w) acc += s_warp[w];
  const unsigned below = (1u << lane) - 1u;
#pragma unroll
  for (int k = 0; k < per32; ++k) {
    m.pos[wbase + k * 32 + lane] = static_cast<uint16_t>(acc + __popc(flags[k] & below));
    acc += __popc(flags[k]);
  }
  if (threadIdx.x < 32) {  // warp-wide decoupled look-back: this bucket's output offset
    uint32_t total = 0;
    for (int w = 0; w < 16; ++w) total += s_warp[w];
    constexpr unsigned long long kCount = 1ULL << 62, kPrefix = 2ULL << 62, kVal = (1ULL << 62) - 1;
    unsigned long long prefix = 0;
    if (bucket == 0) {
      if (lane == 0) atomicExch(&state[0], kPrefix | total);
    } else {
      if (lane == 0) atomicExch(&state[bucket], kCount | total);
      // 32 predecessors per round (one lane each, nearest first): sum back to the nearest one
      // that has published its inclusive prefix; a round with a predecessor still folding (flag
      // 0) before that point is re-read (it runs: it claimed its ticket first). A one-thread walk
      // read one predecessor per L2 round trip (~600 CTAs in flight: the emit's top stall).
      for (int64_t j = static_cast<int64_t>(bucket) - 1;;) {
        const int64_t idx = j - lane;
        const unsigned long long v = idx >= 0 ? atomicAdd(&state[idx], 0ULL) : kPrefix;
        const unsigned f = static_cast<unsigned>(v >> 62);
        const unsigned pm = __ballot_sync(0xffffffffu, f == 2), zm = __ballot_sync(0xffffffffu, f == 0);
        const int fp = pm ? __ffs(pm) - 1 : 32;  // nearest lane holding a prefix
        const unsigned need = fp < 31 ? (2u << fp) - 1u : 0xffffffffu;
        if (zm & need) continue;
        unsigned long long c = lane <= fp ? (v & kVal) : 0ULL;
        for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
        prefix += c;
        if (fp < 32) break;
        j -= 32;
      }
      if (lane == 0) atomicExch(&state[bucket], kPrefix | (prefix + total));
    }
    if (lane == 0) s_base = prefix;
  }
  __syncthreads();
  // rows in key order: walk the key-bitmap words covering the bucket's slots
  const unsigned long long* bits = reinterpret_cast<const unsigned long long*>(t.kbits);
  const uint64_t obase = s_base;
  const bool st32 = nc == 4 && (reinterpret_cast<uintptr_t>(out) & 31) == 0;
  for (uint64_t w = first_word[bucket] + threadIdx.x; w < nwords; w += blockDim.x) {
    uint64_t s = t.krank[w];
    if (s >= s_end) break;
    unsigned long long mb = bits[w];
    while (mb) {
      const int bit = __ffsll(static_cast<long long>(mb)) - 1;
      mb &= mb - 1;
      const uint64_t slot = s++;
      if (slot < s0) continue;
      if (slot >= s_end) break;
      const int i = static_cast<int>(slot - s0);
      const uint64_t hits = m.hits[i];
      if (!hits) continue;
      const uint64_t key = static_cast<uint64_t>(t.kmin) + (w << 6) + bit;
      auto col = [&](int k) -> uint64_t {
        const int kind = ec.kind[k], j = ec.idx[k];
        if (kind == 0) return key;
        if (kind == 1) return hits;  // unique build keys: multiplicity 1
        if (kind == 2)
          return ((static_cast<uint64_t>(m.hi[j * kBucketSlots + i]) << 32) | m.lo[j * kBucketSlots + i]) +
                 hits * static_cast<uint64_t>(b.min[j]);
        const uint64_t c = t.cold[slot * t.cw + 1 + j];
        return t.bs_float[j] ? static_cast<uint64_t>(__double_as_longlong(
                                   static_cast<double>(hits) * __longlong_as_double(static_cast<long long>(c))))
                             : hits * c;
      };
      uint64_t* row = out + (obase + m.pos[i]) * nc;
      if (st32)
        st256(row, col(0), col(1), col(2), col(3));
      else
        for (int k = 0; k < nc; ++k) row[k] = col(k);
    }
  }
  __syncthreads();  // smem and s_bucket are reused by the next bucket
  }
}

void launch_bucket_emit(const AggTableDev& t, const BucketDev& b, uint64_t nbuckets, uint64_t nslots,
                        unsigned long long* state, unsigned int* ticket, uint32_t* first_word, int nc,
                        const int32_t* col_kind, const int32_t* col_idx, uint64_t* out_rows, void* stream) {
  if (nbuckets == 0) return;
  const uint64_t nwords = (t.krange + 63) / 64;
  count_launch();
  k_bucket_words<<<grid_for(nwords, 256), 256, 0, S(stream)>>>(t, nwords, nslots, first_word);
  EmitCols ec{};
  for (int k = 0; k < nc; ++k) {
    ec.kind[k] = col_kind[k];
    ec.idx[k] = col_idx[k];
  }
  const int smem = (1 + 2 * t.nps) * kBucketSlots * 4 + kBucketSlots * 2;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_bucket_emit, cudaFuncAttributeMaxDynamicSharedMemorySize, (1 + 2 * 3) * kBucketSlots * 4 + kBucketSlots * 2);
    attr = true;
  }
  count_launch();
  cudaMemsetAsync(state, 0, nbuckets * sizeof(unsigned long long), S(stream));
  cudaMemsetAsync(ticket, 0, sizeof(unsigned int), S(stream));
  int per_sm = 0, sms = 148, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_bucket_emit, 512, smem);
  const int resident = sms * std::max(per_sm, 1);
  const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(nbuckets, static_cast<uint64_t>(resident)));
  k_bucket_emit<<<grid, 512, smem, S(stream)>>>(t, b, nslots, nwords, state, ticket, first_word, nc, ec, out_rows,
                                                 nbuckets);
}

/// Destination histogram of n keys (partition_of, hashing.hpp:35-37): one shared atomic per
/// (warp, destination) from __match_any_sync groups, one global atomic per (block, destination).
__global__ void k_part_hist(const uint64_t* __restrict__ keys, uint64_t n, int nparts, unsigned long long* counts) {
  __shared__ unsigned long long s_cnt[kMaxParts];
  for (int d = threadIdx.x; d < nparts; d += blockDim.x) s_cnt[d] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  for (uint64_t base = blockIdx.x * static_cast<uint64_t>(blockDim.x); base < n;
       base += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t i = base + threadIdx.x;
    const uint32_t d = i < n ? part_of(keys[i], static_cast<uint32_t>(nparts)) : 0xffffffffu;
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    if (d != 0xffffffffu && lane == __ffs(peers) - 1) atomicAdd(&s_cnt[d], static_cast<unsigned long long>(__popc(peers)));
  }
  __syncthreads();
  for (int d = threadIdx.x; d < nparts; d += blockDim.x)
    if (s_cnt[d]) atomicAdd(&counts[d], s_cnt[d]);
}
void launch_part_hist(const uint64_t* keys, uint64_t n, int nparts, unsigned long long* counts, void* stream) {
  if (n == 0) return;
  count_launch();
  k_part_hist<<<grid_for(n, 256), 256, 0, S(stream)>>>(keys, n, nparts, counts);
}

/// out[0] = min, out[1] = max of n signed keys (out preset to {INT64_MAX, INT64_MIN}).
__global__ void k_minmax_i64(const uint64_t* keys, uint64_t n, long long* out) {
  long long lo = LLONG_MAX, hi = LLONG_MIN;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const long long k = static_cast<long long>(keys[i]);
    lo = min(lo, k);
    hi = max(hi, k);
  }
  for (int o = 16; o > 0; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(out, lo);
    atomicMax(out + 1, hi);
  }
}
void launch_minmax_i64(const uint64_t* keys, uint64_t n, long long* out, void* stream) {
  if (n == 0) return;
  count_launch();
  k_minmax_i64<<<grid_for(n, 256), 256, 0, S(stream)>>>(keys, n, out);
}
/// Membership bitmap of keys - bmin; *dup = 1 when a key repeats.
__global__ void k_bitmap_set(const uint64_t* keys, uint64_t n, int64_t bmin, uint32_t* bitmap, unsigned int* dup) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t d = keys[i] - static_cast<uint64_t>(bmin);
    const uint32_t bit = 1u << (d & 31);
    if (atomicOr(bitmap + (d >> 5), bit) & bit) *dup = 1u;
  }
}

/// Hot slots of the rank-indexed table in slot (= key) order: one thread per 64-bit word of the
/// key bitmap writes {key, 0...} for each of its set bits at consecutive slots from krank[w].
__global__ void k_rank_hot(AggTableDev t, uint64_t nwords) {
  const unsigned long long* bits = reinterpret_cast<const unsigned long long*>(t.kbits);
  for (uint64_t w = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; w < nwords;
       w += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    unsigned long long m = bits[w];
    uint64_t r = t.krank[w];
    const uint64_t base = static_cast<uint64_t>(t.kmin) + (w << 6);
    while (m) {
      const int b = __ffsll(static_cast<long long>(m)) - 1;
      m &= m - 1;
      uint64_t* h = t.hot + r * t.hw;
      st256(h, base + b, 0, 0, 0);
      for (int k = 4; k < t.hw; k += 4) st256(h + k, 0, 0, 0, 0);
      ++r;
    }
  }
}

/// Rank-indexed aggregation table build (unique dense build keys, one GPU): row i of the build
/// side lands in the slot of its key's rank - plain stores, no CAS, every slot written once.
/// Build-side double sums are stored as 0.0 + v (the value a hash-table insert accumulates).
template <bool kHot>
__global__ void k_rank_build(AggTableDev t, const uint64_t* __restrict__ keys, RankSums bs, uint64_t n) {
  const uint64_t tid = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  for (uint64_t i = tid; i < n; i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t key = keys[i];
    uint64_t cv[2 * kMaxSums + 2];
    cv[0] = 0;
#pragma unroll
    for (int b = 0; b < kMaxSums; ++b) {
      if (b >= t.nbs) break;
      const uint64_t v = bs.col[b][i];
      cv[1 + b] = t.bs_float[b]
                      ? static_cast<uint64_t>(__double_as_longlong(0.0 + __longlong_as_double(static_cast<long long>(v))))
                      : v;
    }
    const uint64_t r = agg_rank_slot(t, key);
    if (kHot) {
      uint64_t* h = t.hot + r * t.hw;
      if (t.hw % 4 == 0) {  // whole 32-byte sectors per store: no partial-sector fills from DRAM
        st256(h, key, 0, 0, 0);
        for (int k = 4; k < t.hw; k += 4) st256(h + k, 0, 0, 0, 0);
      } else {
        *reinterpret_cast<ulonglong2*>(h) = make_ulonglong2(key, 0ULL);
      }
    }
    uint64_t* c = t.cold + r * t.cw;  // cw is a multiple of 4 here
#pragma unroll
    for (int k = 0; k < 2 * kMaxSums + 2; k += 4) {
      if (k >= t.cw) break;
      auto w = [&](int j) { return j <= t.nbs ? cv[j] : 0ULL; };
      st256(c + k, w(k), w(k + 1), w(k + 2), w(k + 3));
    }
  }
}

void launch_rank_build(const AggTableDev& t, const uint64_t* keys, const RankSums& bs, uint64_t n, bool first,
                       bool write_hot, void* stream) {
  // The hot slots are written in slot order from the key bitmap (k_rank_hot, sequential stores)
  // and the row-ordered build pass writes only the cold slots: the build rows arrive in scan
  // order, not key order, so hot-slot stores by row were scattered (SF100 N=1: one 0.60 ms pass
  // -> 0.09 + 0.30 ms). Without build-side sums the cold slots hold nothing but the multiplicity
  // m - 1 = 0 of unique keys, which nothing reads (emit reads cold only for duplicates and the
  // spill slot), so that pass is skipped (Q3: -0.25 ms). PSG_RANK_HOT_SEQ=0: one row-ordered pass
  // for both. `first`: this call also writes the hot slots and clears the (never occupied) spill
  // slot; later calls (more build segments at N > 1) only their rows' cold slots.
  static const bool hot_seq = [] {
    const char* e = std::getenv("PSG_RANK_HOT_SEQ");
    return !(e && e[0] == '0');
  }();
  const uint64_t spill = t.mask + 1;
  if (first) {
    cudaMemsetAsync(t.hot + spill * t.hw, 0, t.hw * sizeof(uint64_t), S(stream));
    cudaMemsetAsync(t.cold + spill * t.cw, 0, t.cw * sizeof(uint64_t), S(stream));
  }
  if (!write_hot) {  // bucketed aggregation: the hot table is zeroed, keys come from the bitmap
    if (t.nbs > 0 && n > 0) {
      count_launch();
      k_rank_build<false><<<grid_for(n, 256), 256, 0, S(stream)>>>(t, keys, bs, n);
    }
  } else if (hot_seq && t.hw % 4 == 0) {
    if (first) {
      const uint64_t nw = (t.krange + 63) / 64;
      count_launch();
      k_rank_hot<<<grid_for(std::max<uint64_t>(nw, 1), 256), 256, 0, S(stream)>>>(t, nw);
    }
    if (t.nbs > 0 && n > 0) {
      count_launch();
      k_rank_build<false><<<grid_for(n, 256), 256, 0, S(stream)>>>(t, keys, bs, n);
    }
  } else if (n > 0) {
    count_launch();
    k_rank_build<true><<<grid_for(n, 256), 256, 0, S(stream)>>>(t, keys, bs, n);
  }
}

/// Bloom bits of a key column (the semi-join filter of the received build rows, set ahead of the
/// table insert so the probe side can start screening while the insert runs).
__global__ void k_bloom_keys(const uint64_t* __restrict__ keys, uint64_t n, uint32_t* bloom, int shift) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t key = keys[i];
    if (key == kEmptyKey) continue;  // null keys are never screened
    const uint64_t h2 = key * kBloomMul;
    atomicOr(bloom + (h2 >> shift), bloom_bits(h2, shift));
  }
}

void launch_bloom_keys(const uint64_t* keys, uint64_t n, uint32_t* bloom, int shift, void* stream) {
  if (n == 0) return;
  count_launch();
  k_bloom_keys<<<grid_for(n, 256), 256, 0, S(stream)>>>(keys, n, bloom, shift);
}

void launch_bitmap_set(const uint64_t* keys, uint64_t n, int64_t bmin, uint32_t* bitmap, unsigned int* dup, void* stream) {
  if (n == 0) return;
  count_launch();
  k_bitmap_set<<<grid_for(n, 256), 256, 0, S(stream)>>>(keys, n, bmin, bitmap, dup);
}

// --------------------------------------------------------------------------- result emission
/// counter[0] = groups, counter[1] = min, counter[2] = max of the sign-flipped keys (the sort
/// then only needs the bits where min and max differ: all keys share the bits above). Each block
/// compacts a contiguous range of 4096 slots with one global atomic (block prefix in smem).
constexpr int kCompactSpan = 4096;
__global__ void __launch_bounds__(256) k_agg_compact(AggTableDev t, uint64_t nslots, uint64_t* out_keys,
                                                     unsigned long long* out_slots, unsigned long long* counter) {
  __shared__ uint32_t s_cnt[kCompactSpan / 32];
  __shared__ unsigned long long s_base;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  unsigned long long lo = ~0ULL, hi = 0;
  for (uint64_t span = blockIdx.x * static_cast<uint64_t>(kCompactSpan); span < nslots;
       span += static_cast<uint64_t>(gridDim.x) * kCompactSpan) {
    constexpr int PER = kCompactSpan / 256;  // slots per thread, warp-strided
    bool take[PER];
    uint64_t key[PER];
    unsigned bal[PER];
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const uint64_t s = span + (warp * PER + k) * 32 + lane;
      take[k] = false;
      key[k] = 0;
      if (s < nslots) {
        const ulonglong2 kh = *reinterpret_cast<const ulonglong2*>(t.hot + s * t.hw);  // {key, hits}
        key[k] = kh.x;
        const bool occupied = (s == nslots - 1) ? (t.cold[s * t.cw] > 0) : (kh.x != kEmptyKey);
        take[k] = occupied && kh.y > 0;
      }
      bal[k] = __ballot_sync(0xffffffffu, take[k]);
      if (lane == 0) s_cnt[warp * PER + k] = __popc(bal[k]);
    }
    __syncthreads();
    if (warp == 0) {  // exclusive scan of the 128 per-(warp,k) counts, 4 per lane
      uint32_t c[4], sum = 0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        c[q] = s_cnt[lane * 4 + q];
        sum += c[q];
      }
      uint32_t incl = sum;
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      uint32_t run = incl - sum;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t x = c[q];
        s_cnt[lane * 4 + q] = run;
        run += x;
      }
      const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
      if (lane == 31) s_base = total ? atomicAdd(counter, static_cast<unsigned long long>(total)) : 0ULL;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      if (!take[k]) continue;
      const uint64_t s = span + (warp * PER + k) * 32 + lane;
      const uint64_t pos = s_base + s_cnt[warp * PER + k] + __popc(bal[k] & ((1u << lane) - 1u));
      const uint64_t fk = key[k] ^ 0x8000000000000000ULL;  // signed order under an unsigned radix sort
      out_keys[pos] = fk;
      out_slots[pos] = s;
      lo = min(lo, static_cast<unsigned long long>(fk));
      hi = max(hi, static_cast<unsigned long long>(fk));
    }
    __syncthreads();
  }
  for (int o = 16; o > 0; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if (lane == 0 && hi >= lo) {
    atomicMin(counter + 1, lo);
    atomicMax(counter + 2, hi);
  }
}
void launch_agg_compact(const AggTableDev& t, uint64_t cap, uint64_t* out_keys, unsigned long long* out_slots,
                        unsigned long long* counter, void* stream) {
  count_launch();
  uint64_t blocks = (cap + 1 + kCompactSpan - 1) / kCompactSpan;
  const uint64_t maxb = static_cast<uint64_t>(sm_count()) * 8;
  if (blocks > maxb) blocks = maxb;
  k_agg_compact<<<static_cast<unsigned>(blocks), 256, 0, S(stream)>>>(t, cap + 1, out_keys, out_slots, counter);
}

// ---- dense finalisation: when the group keys span a range R not much larger than the group
// count, the output position of a group is its key's rank in a bitmap of present keys
// (prefix popcount), so rows are written straight from a sequential table pass - no sort, no
// gather through a sorted slot list.
__global__ void __launch_bounds__(256) k_agg_range(AggTableDev t, uint64_t nslots, unsigned long long* counter) {
  unsigned long long lo = ~0ULL, hi = 0, n = 0;
  for (uint64_t s = blockIdx.x * 256ULL + threadIdx.x; s < nslots; s += gridDim.x * 256ULL) {
    const ulonglong2 kh = *reinterpret_cast<const ulonglong2*>(t.hot + s * t.hw);
    const bool occupied = (s == nslots - 1) ? (t.cold[s * t.cw] > 0) : (kh.x != kEmptyKey);
    if (occupied && kh.y > 0) {
      const unsigned long long fk = kh.x ^ 0x8000000000000000ULL;
      lo = min(lo, fk);
      hi = max(hi, fk);
      ++n;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    n += __shfl_xor_sync(0xffffffffu, n, o);
  }
  if ((threadIdx.x & 31) == 0 && n) {
    atomicAdd(counter, n);
    atomicMin(counter + 1, lo);
    atomicMax(counter + 2, hi);
  }
}
__global__ void __launch_bounds__(256) k_agg_mark(AggTableDev t, uint64_t nslots, unsigned long long fmin,
                                                  unsigned long long* bitmap) {
  for (uint64_t s = blockIdx.x * 256ULL + threadIdx.x; s < nslots; s += gridDim.x * 256ULL) {
    const ulonglong2 kh = *reinterpret_cast<const ulonglong2*>(t.hot + s * t.hw);
    const bool occupied = (s == nslots - 1) ? (t.cold[s * t.cw] > 0) : (kh.x != kEmptyKey);
    if (occupied && kh.y > 0) {
      const uint64_t b = (kh.x ^ 0x8000000000000000ULL) - fmin;
      atomicOr(bitmap + (b >> 6), 1ULL << (b & 63));
    }
  }
}
__global__ void k_popc64(const unsigned long long* bitmap, uint64_t nwords, uint32_t* out) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < nwords;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    out[i] = __popcll(bitmap[i]);
}

__global__ void k_agg_emit(AggTableDev t, const uint64_t* keys, const unsigned long long* slots, uint64_t n, int nc,
                           EmitCols ec, uint64_t* out) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t s = slots[i];
    const uint64_t* h = t.hot + s * t.hw;
    const uint64_t* c = t.cold + s * t.cw;
    const uint64_t hits = agg_hits(t, h), m = (t.dups == nullptr || *t.dups != 0 || s == t.mask + 1) ? agg_mult(t, s) : 1;
    uint64_t* row = out + i * nc;
    for (int k = 0; k < nc; ++k) {
      const int kind = ec.kind[k], j = ec.idx[k];
      uint64_t v = 0;
      if (kind == 0) {
        v = keys[i] ^ 0x8000000000000000ULL;
      } else if (kind == 1) {
        v = hits * m;
      } else if (kind == 2) {  // probe-side sum: each probe row pairs with m build rows
        v = t.ps_float[j] ? static_cast<uint64_t>(__double_as_longlong(
                                static_cast<double>(m) * __longlong_as_double(static_cast<long long>(h[2 + j]))))
                          : m * agg_psum(t, h, j, hits);
      } else {  // build-side sum: each matched probe row adds the key's build-side total
        v = t.bs_float[j] ? static_cast<uint64_t>(__double_as_longlong(
                                static_cast<double>(hits) * __longlong_as_double(static_cast<long long>(c[1 + j]))))
                          : hits * c[1 + j];
      }
      row[k] = v;
    }
  }
}
/// Dense emit: one pass over the table; row of the group with flipped key fk goes to
/// prefix[w] + popc(bitmap[w] & below) with w, b = (fk - fmin) / 64, % 64.
__global__ void __launch_bounds__(256) k_agg_emit_dense(AggTableDev t, uint64_t nslots, unsigned long long fmin,
                                                        const unsigned long long* bitmap, const uint32_t* prefix, int nc,
                                                        EmitCols ec, uint64_t* out) {
  const bool dups = t.dups == nullptr || *t.dups != 0;
  const bool st32 = (nc & 3) == 0 && (reinterpret_cast<uintptr_t>(out) & 31) == 0;
  for (uint64_t s = blockIdx.x * 256ULL + threadIdx.x; s < nslots; s += gridDim.x * 256ULL) {
    const uint64_t* h = t.hot + s * t.hw;
    const ulonglong2 kh = *reinterpret_cast<const ulonglong2*>(h);
    const bool spill = s == nslots - 1;
    const bool occupied = spill ? (t.cold[s * t.cw] > 0) : (kh.x != kEmptyKey);
    if (!occupied || kh.y == 0) continue;
    const uint64_t b = (kh.x ^ 0x8000000000000000ULL) - fmin;
    const uint64_t w = b >> 6;
    const uint64_t pos = prefix[w] + __popcll(bitmap[w] & ((1ULL << (b & 63)) - 1ULL));
    const uint64_t* c = t.cold + s * t.cw;
    const uint64_t hits = t.npacked ? (kh.y & t.hits_mask) : kh.y, m = (spill || dups) ? agg_mult(t, s) : 1;
    uint64_t* row = out + pos * nc;
    uint64_t vals[2 * kMaxSums + 2];
#pragma unroll
    for (int k = 0; k < 2 * kMaxSums + 2; ++k) {
      if (k >= nc) break;
      const int kind = ec.kind[k], j = ec.idx[k];
      uint64_t v;
      if (kind == 0) {
        v = kh.x;
      } else if (kind == 1) {
        v = hits * m;
      } else if (kind == 2) {
        v = t.ps_float[j] ? static_cast<uint64_t>(__double_as_longlong(
                                static_cast<double>(m) * __longlong_as_double(static_cast<long long>(h[2 + j]))))
                          : m * agg_psum(t, h, j, hits);
      } else {
        v = t.bs_float[j] ? static_cast<uint64_t>(__double_as_longlong(
                                static_cast<double>(hits) * __longlong_as_double(static_cast<long long>(c[1 + j]))))
                          : hits * c[1 + j];
      }
      vals[k] = v;
    }
    // rows land at random positions (hashed table): whole 32-byte stores where rows are whole
    // sectors (no partial-sector fills from DRAM), else 16-byte stores
    if (st32) {
#pragma unroll
      for (int k = 0; k < 2 * kMaxSums + 2; k += 4) {
        if (k >= nc) break;
        st256(row + k, vals[k], vals[k + 1], vals[k + 2], vals[k + 3]);
      }
    } else if ((nc & 1) == 0) {
#pragma unroll
      for (int k = 0; k < 2 * kMaxSums + 2; k += 2) {
        if (k >= nc) break;
        *reinterpret_cast<ulonglong2*>(row + k) = make_ulonglong2(vals[k], vals[k + 1]);
      }
    } else {
#pragma unroll
      for (int k = 0; k < 2 * kMaxSums + 2; ++k) {
        if (k >= nc) break;
        row[k] = vals[k];
      }
    }
  }
}

void launch_agg_range(const AggTableDev& t, uint64_t cap, unsigned long long* counter, void* stream) {
  count_launch();
  k_agg_range<<<sm_count() * 8, 256, 0, S(stream)>>>(t, cap + 1, counter);
}
void launch_agg_mark(const AggTableDev& t, uint64_t cap, uint64_t fmin, unsigned long long* bitmap, void* stream) {
  count_launch();
  k_agg_mark<<<sm_count() * 8, 256, 0, S(stream)>>>(t, cap + 1, fmin, bitmap);
}
void launch_popc64(const unsigned long long* bitmap, uint64_t nwords, uint32_t* out, void* stream) {
  count_launch();
  k_popc64<<<grid_for(nwords, 256), 256, 0, S(stream)>>>(bitmap, nwords, out);
}
void launch_agg_emit_dense(const AggTableDev& t, uint64_t cap, uint64_t fmin, const unsigned long long* bitmap,
                           const uint32_t* prefix, int nc, const int32_t* col_kind, const int32_t* col_idx,
                           uint64_t* out_rows, void* stream) {
  EmitCols ec{};
  for (int k = 0; k < nc; ++k) {
    ec.kind[k] = col_kind[k];
    ec.idx[k] = col_idx[k];
  }
  count_launch();
  k_agg_emit_dense<<<sm_count() * 8, 256, 0, S(stream)>>>(t, cap + 1, fmin, bitmap, prefix, nc, ec, out_rows);
}

void launch_agg_emit(const AggTableDev& t, const uint64_t* sorted_keys, const unsigned long long* sorted_slots,
                     uint64_t n, int nc, const int32_t* col_kind, const int32_t* col_idx, uint64_t* out_rows,
                     void* stream) {
  if (n == 0) return;
  EmitCols ec{};
  for (int k = 0; k < nc; ++k) {
    ec.kind[k] = col_kind[k];
    ec.idx[k] = col_idx[k];
  }
  count_launch();
  k_agg_emit<<<grid_for(n, 256), 256, 0, S(stream)>>>(t, sorted_keys, sorted_slots, n, nc, ec, out_rows);
}

size_t sort_pairs_i64(const uint64_t* keys_in, uint64_t* keys_out, const unsigned long long* v_in,
                      unsigned long long* v_out, uint64_t n, int end_bit, void* tmp, size_t tmp_bytes, void* stream) {
  size_t bytes = tmp_bytes;
  cub::DeviceRadixSort::SortPairs(tmp, bytes, reinterpret_cast<const unsigned long long*>(keys_in),
                                  reinterpret_cast<unsigned long long*>(keys_out), v_in, v_out,
                                  static_cast<int64_t>(n), 0, end_bit, S(stream));
  if (tmp) count_launch();
  return bytes;
}
size_t sort_pairs_u32(const uint32_t* keys_in, uint32_t* keys_out, const uint32_t* v_in, uint32_t* v_out, uint64_t n,
                      int end_bit, void* tmp, size_t tmp_bytes, void* stream) {
  size_t bytes = tmp_bytes;
  cub::DeviceRadixSort::SortPairs(tmp, bytes, keys_in, keys_out, v_in, v_out, static_cast<int64_t>(n), 0, end_bit,
                                  S(stream));
  if (tmp) count_launch();
  return bytes;
}

__global__ void k_iota(uint32_t* out, uint64_t n) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    out[i] = static_cast<uint32_t>(i);
}
void launch_iota_u32(uint32_t* out, uint64_t n, void* stream) {
  if (n == 0) return;
  count_launch();
  k_iota<<<grid_for(n, 256), 256, 0, S(stream)>>>(out, n);
}

__global__ void k_rows_from_cols(ColPtrs in, int nc, uint64_t n, uint64_t* out) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    for (int c = 0; c < nc; ++c) out[i * nc + c] = in.p[c][i];
}
void launch_rows_from_cols(const uint64_t* const* cols, int nc, uint64_t n, uint64_t* out_rows, void* stream) {
  if (n == 0 || nc == 0) return;
  ColPtrs pc{};
  for (int c = 0; c < nc; ++c) pc.p[c] = cols[c];
  count_launch();
  k_rows_from_cols<<<grid_for(n, 256), 256, 0, S(stream)>>>(pc, nc, n, out_rows);
}

}  // namespace psg
