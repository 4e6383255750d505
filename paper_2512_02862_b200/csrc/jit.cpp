// Query compilation: the fused scan kernel specialised per plan program with NVRTC for sm_100a.
//
// k_scan (kernels.cu) interprets a ScanProgram at run time: register indices, atom operators,
// join chains and sinks are data, which costs ~250 warp instructions per row (ncu, profiles/).
// Here the same program is emitted as straight-line CUDA C++ — every column lives in named
// registers, operators are inlined, loops over columns/atoms/sums disappear — and compiled once
// per distinct program *structure* (literals, table pointers and outputs stay in the kernel's
// __grid_constant__ ScanProgram, so the cache hits across literal changes and queries). The
// generated kernel shares device_common.cuh (layout + hashing) with the nvcc-built kernels.
// Fallback when NVRTC is unavailable: the interpreter k_scan (still GPU; there is no CPU path).
#include <cuda_runtime.h>
#include <nvrtc.h>
#include <unistd.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <sstream>
#include <cstring>
#include <string>
#include <vector>

#include "common.hpp"
#include "jit.hpp"
#include "kernels.cuh"

namespace psg {

namespace {
#include "_gen_device_common.inc"  // kDeviceCommonSrc: device_common.cuh verbatim (build.py)

struct Compiled {
  cudaLibrary_t lib = nullptr;
  cudaKernel_t kern = nullptr;
  int block = kBlock;  // threads per CTA (jit_block)
  int smem = 0;        // dynamic shared memory per CTA (the staged probe's ring)
  int per_sm = 1;
  bool ok = false;
};

std::mutex g_mu;
std::map<std::pair<int, std::string>, Compiled> g_cache;
double g_compile_s = 0;
uint64_t g_compiles = 0;

bool jit_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("PSG_JIT");
    return !(e && e[0] == '0');
  }();
  return on;
}

std::string V(int reg) { return "v" + std::to_string(reg); }

const char* op_str(int op) {
  switch (op) {
    case 0: return "<";
    case 1: return "<=";
    case 2: return "==";
    case 3: return "!=";
    case 4: return ">=";
    default: return ">";
  }
}

/// Emits `for r: if (pass & bit) vC[r] = load(col c of the tile)` for columns [lo, hi).
void emit_loads(std::ostringstream& s, int lo, int hi) {
  for (int c = lo; c < hi; ++c) {
    s << "    { const uint64_t* col = reinterpret_cast<const uint64_t*>(__shfl_sync(0xffffffffu, "
         "reinterpret_cast<unsigned long long>(cur_col), " << c << ")) + row0 + wrow;\n"
      << "#pragma unroll\n      for (int r = 0; r < R; ++r) if (pass & (1u << r)) " << V(c)
      << "[r] = __ldcs(reinterpret_cast<const unsigned long long*>(col + r * 32));\n    }\n";
  }
}

/// Semi-join screen against the all-gathered per-owner Bloom filters (local copy).
void emit_semi(std::ostringstream& s, const ScanProgram& P) {
  s << "    { uint32_t bw[R], bm[R];\n"
    << "#pragma unroll\n      for (int r = 0; r < R; ++r) { bw[r] = bm[r] = 0; const uint64_t key = " << V(P.semi_key_reg)
    << "[r];\n        if ((pass & (1u << r)) && key != kEmptyKey) { const uint64_t h2 = key * kBloomMul;\n"
    << "          const uint32_t d = part_of(key, static_cast<uint32_t>(P.nparts));\n"
    << "          bm[r] = bloom_bits(h2, P.semi_shift); bw[r] = ldg_keep_u32(P.semi_bloom + d * P.semi_words + (h2 >> P.semi_shift), pol_keep); } }\n"
    << "#pragma unroll\n      for (int r = 0; r < R; ++r) if ((pass & (1u << r)) && (bw[r] & bm[r]) != bm[r]) pass &= ~(1u << r);\n    }\n";
}

/// Fused build over NVLink: each key is inserted straight into its owner's (peer-mapped) table.
void emit_remote_build(std::ostringstream& s, const ScanProgram& P) {
  const int hw = P.agg.hw, cw = P.agg.cw;
  s << "    { const AggTableDev& T = P.agg;\n      uint64_t sl[R]; unsigned long long pv[R];\n"
    << "#pragma unroll\n      for (int r = 0; r < R; ++r) { sl[r] = 0; pv[r] = kEmptyKey; if (!(pass & (1u << r))) continue;\n"
    << "        const uint64_t key = " << V(P.key_reg) << "[r];\n"
    << "        if (key == kEmptyKey) { sl[r] = T.mask + 1; continue; }\n"
    << "        uint64_t* hot = P.peers[part_of(key, static_cast<uint32_t>(P.nparts))].hot;\n"
    << "        sl[r] = slot_of(key, T.shift);\n"
    << "        pv[r] = atomicCAS_system(reinterpret_cast<unsigned long long*>(hot + sl[r] * " << hw << "), kEmptyKey, key); }\n"
    << "#pragma unroll\n      for (int r = 0; r < R; ++r) { if (!(pass & (1u << r))) continue;\n"
    << "        const uint64_t key = " << V(P.key_reg) << "[r];\n"
    << "        const AggPeer pe = P.peers[part_of(key, static_cast<uint32_t>(P.nparts))];\n"
    << "        uint64_t sx = sl[r]; bool dup = pv[r] == key;\n"
    << "        if (pv[r] != kEmptyKey && pv[r] != key) {\n"
    << "          sx = (sx + 1) & T.mask;\n"
    << "          while (true) { const unsigned long long prev = atomicCAS_system(reinterpret_cast<unsigned long long*>(pe.hot + sx * "
    << hw << "), kEmptyKey, key);\n"
    << "            if (prev == kEmptyKey || prev == key) { dup = prev == key; break; } sx = (sx + 1) & T.mask; } }\n"
    << "        unsigned long long* cold = reinterpret_cast<unsigned long long*>(pe.cold + sx * " << cw << ");\n"
    << "        if (sx == T.mask + 1 || dup) atomicAdd_system(cold, 1ULL);\n"
    << "        else if (pe.bloom != nullptr) { const uint64_t h2 = key * kBloomMul;\n"
    << "          atomicOr_system(pe.bloom + (h2 >> T.bloom_shift), bloom_bits(h2, T.bloom_shift)); }\n";
  for (int bb = 0; bb < P.n_sum; ++bb) {
    if (P.agg.bs_float[bb])
      s << "        atomicAdd_system(reinterpret_cast<double*>(cold + " << 1 + bb << "), __longlong_as_double(static_cast<long long>("
        << V(P.sum_reg[bb]) << "[r])));\n";
    else
      s << "        atomicAdd_system(cold + " << 1 + bb << ", static_cast<unsigned long long>(" << V(P.sum_reg[bb]) << "[r]));\n";
  }
  s << "      }\n    }\n";
}

/// Fused probe + aggregation over NVLink: semi-join screen locally, then probe the owner's
/// (peer-mapped) table and accumulate in its slot with system-scope atomics.
void emit_remote_probe(std::ostringstream& s, const ScanProgram& P) {
  const int hw = P.agg.hw, cw = P.agg.cw;
  if (P.semi_bloom) emit_semi(s, P);
  s << "    { const AggTableDev& T = P.agg;\n      uint64_t sl[R], k0[R]; uint64_t* hb[R];\n"
    << "#pragma unroll\n      for (int r = 0; r < R; ++r) { sl[r] = ~0ULL; k0[r] = 0; hb[r] = nullptr; if (!(pass & (1u << r))) continue;\n"
    << "        const uint64_t key = " << V(P.key_reg) << "[r];\n"
    << "        const AggPeer pe = P.peers[part_of(key, static_cast<uint32_t>(P.nparts))];\n        hb[r] = pe.hot;\n"
    << "        if (key == kEmptyKey) { if (pe.cold[(T.mask + 1) * " << cw << "] == 0) pass &= ~(1u << r); else sl[r] = T.mask + 1; }\n"
    << "        else { sl[r] = slot_of(key, T.shift); k0[r] = hb[r][sl[r] * " << hw << "]; } }\n"
    << "#pragma unroll\n      for (int r = 0; r < R; ++r) { if (!(pass & (1u << r)) || sl[r] == T.mask + 1) continue;\n"
    << "        const uint64_t key = " << V(P.key_reg) << "[r]; uint64_t sx = sl[r], kk = k0[r];\n"
    << "        while (kk != key && kk != kEmptyKey) { sx = (sx + 1) & T.mask; kk = hb[r][sx * " << hw << "]; }\n"
    << "        if (kk != key) pass &= ~(1u << r); else sl[r] = sx; }\n";
  emit_loads(s, P.n_early, P.n_in);
  s << "#pragma unroll\n      for (int r = 0; r < R; ++r) { if (!(pass & (1u << r))) continue;\n"
    << "        unsigned long long* h = reinterpret_cast<unsigned long long*>(hb[r] + sl[r] * " << hw << ");\n"
    << "        atomicAdd_system(h + 1, 1ULL);\n";
  for (int p = 0; p < P.n_sum; ++p) {
    if (P.agg.ps_float[p])
      s << "        atomicAdd_system(reinterpret_cast<double*>(h + " << 2 + p << "), __longlong_as_double(static_cast<long long>("
        << V(P.sum_reg[p]) << "[r])));\n";
    else
      s << "        atomicAdd_system(h + " << 2 + p << ", static_cast<unsigned long long>(" << V(P.sum_reg[p]) << "[r]));\n";
  }
  s << "      }\n    }\n";
}

}  // namespace

/// Value written to materialised output column o of row r: the register, or with pack_n > 0
/// (one output column) the bit-packed word of the pack registers.
std::string out_value(const ScanProgram& P, int o) {
  if (P.pack_n == 0) return V(P.out_reg[o]) + "[r]";
  std::string e;
  for (int k = 0; k < P.pack_n; ++k) {
    if (k) e += " | ";
    e += "((" + V(P.pack_reg[k]) + "[r] - static_cast<uint64_t>(P.pack_min[" + std::to_string(k) + "])) << P.pack_shift[" +
         std::to_string(k) + "])";
  }
  return "(" + e + ")";
}

/// Accumulation of one matched probe row r into hot slot h (SINK_PROBE and the owner probe):
/// hits (+ packed sums) with one atomicAdd on word 1, unpacked sums on their own words.
void emit_accumulate(std::ostringstream& s, const ScanProgram& P, const char* indent) {
  const bool packed = P.agg.npacked > 0;
  s << indent << "{ unsigned long long inc = 1ULL;\n";
  for (int p = 0; p < P.n_sum; ++p)
    if (packed && !P.agg.ps_float[p] && P.agg.packed_shift[p] >= 0)
      s << indent << "  inc += (static_cast<unsigned long long>(" << V(P.sum_reg[p]) << "[r]) - static_cast<unsigned long long>(T.packed_min["
        << p << "])) << T.packed_shift[" << p << "];\n";
  s << indent << "  atomicAdd(h + 1, inc); }\n";
  for (int p = 0; p < P.n_sum; ++p) {
    if (packed && !P.agg.ps_float[p] && P.agg.packed_shift[p] >= 0) continue;
    if (P.agg.ps_float[p])
      s << indent << "atomicAdd(reinterpret_cast<double*>(h + " << 2 + p << "), __longlong_as_double(static_cast<long long>("
        << V(P.sum_reg[p]) << "[r])));\n";
    else
      s << indent << "atomicAdd(h + " << 2 + p << ", static_cast<unsigned long long>(" << V(P.sum_reg[p]) << "[r]));\n";
  }
}


void emit_rank_tail(std::ostringstream& s, const ScanProgram& P);
/// PSG_BATCH_APPENDS=0: one bucket append (reserve, store) after the other per row.
bool batched_appends() {
  static const bool v = [] {
    const char* e = std::getenv("PSG_BATCH_APPENDS");
    return !(e && e[0] == '0');
  }();
  return v;
}

/// Rank-indexed table probe (SINK_PROBE): the key's 64-bit bitmap word and its block prefix (both
/// L2-resident; one 16-byte {bits, rank} record when krec is set) give membership and the slot at
/// once - no hashing, no collision chain. `late` emits the loads of the non-key columns (for the
/// surviving rows only), then every survivor accumulates into its hot slot.
template <class Late>
void emit_rank_probe(std::ostringstream& s, const ScanProgram& P, Late late) {
  // Screen first (PSG_RANK_SCREEN=0: off): test the 4-byte word of the key bitmap (19 MB vs the
  // rank records' 37 MB at SF100), then read the rank record only for the survivors, with the late
  // columns. SF100 N=1 A/B: probe 3.23 -> 3.19 ms.
  static const bool screen_first = [] {
    const char* e = std::getenv("PSG_RANK_SCREEN");
    return !(e && e[0] == '0');
  }();
  if (screen_first && P.agg.krec != nullptr && P.agg.kbits != nullptr) {
    s << "    { const AggTableDev& T = P.agg; uint32_t gw[R], bb[R], kr[R], sl[R]; unsigned long long kw[R]; uint32_t sel = 0;\n"
      << "#pragma unroll\n      for (int r = 0; r < R; ++r) { const uint64_t key = " << V(P.key_reg) << "[r];\n"
      << "        const uint64_t d = key - static_cast<uint64_t>(T.kmin);\n"
      << "        const bool ok = ((pass >> r) & 1u) && key != kEmptyKey && d < T.krange;\n"
      << "        bb[r] = static_cast<uint32_t>(d & 31); gw[r] = ok ? ldg_keep_u32(T.kbits + (d >> 5), pol_keep) : 0u; }\n"
      << "#pragma unroll\n      for (int r = 0; r < R; ++r) if ((gw[r] >> bb[r]) & 1u) sel |= 1u << r;\n"
      << "#pragma unroll\n      for (int r = 0; r < R; ++r) { kw[r] = 0; kr[r] = 0; if ((sel >> r) & 1u) {\n"
      << "        const uint64_t d = " << V(P.key_reg) << "[r] - static_cast<uint64_t>(T.kmin);\n"
      << "        uint64_t a, b; ldg_keep_v2u64(T.krec + 2 * (d >> 6), pol_keep, a, b); kw[r] = a; kr[r] = static_cast<uint32_t>(b); } }\n"
      << "      pass = sel;\n";
    late();
    s << "#pragma unroll\n      for (int r = 0; r < R; ++r) { const uint32_t d6 = static_cast<uint32_t>((" << V(P.key_reg)
      << "[r] - static_cast<uint64_t>(T.kmin)) & 63);\n"
      << "        sl[r] = kr[r] + static_cast<uint32_t>(__popcll(kw[r] & ((1ULL << d6) - 1ULL))); }\n";
    emit_rank_tail(s, P);
    s << "    }\n";
    return;
  }
  s << "    { const AggTableDev& T = P.agg; uint64_t sl[R]; unsigned long long bw[R]; uint64_t bp[R]; uint32_t bb[R];\n"
    << "#pragma unroll\n      for (int r = 0; r < R; ++r) { bw[r] = 0; bp[r] = 0; bb[r] = 0; const uint64_t key = " << V(P.key_reg) << "[r];\n"
    << "        if ((pass & (1u << r)) && key != kEmptyKey) { const uint64_t d = key - static_cast<uint64_t>(T.kmin);\n"
    << "          if (d < T.krange) { bb[r] = static_cast<uint32_t>(d & 63);\n";
  if (P.agg.krec != nullptr)
    s << "            uint64_t a, b; ldg_keep_v2u64(T.krec + 2 * (d >> 6), pol_keep, a, b); bw[r] = a; bp[r] = b; } } }\n";
  else
    s << "            bw[r] = ldg_keep_u64(reinterpret_cast<const unsigned long long*>(T.kbits) + (d >> 6), pol_keep);\n"
      << "            bp[r] = ldg_keep_u32(T.krank + (d >> 6), pol_keep); } } }\n";
  s << "#pragma unroll\n      for (int r = 0; r < R; ++r) { sl[r] = 0;\n"
    << "        if (!((bw[r] >> bb[r]) & 1ULL)) pass &= ~(1u << r);\n"
    << "        else sl[r] = bp[r] + static_cast<uint64_t>(__popcll(bw[r] & ((1ULL << bb[r]) - 1ULL))); }\n";
  late();
  emit_rank_tail(s, P);
  s << "    }\n";
}

/// Every row still in `pass` accumulates into its rank-table slot sl[r]: one word appended to the
/// slot's bucket (bucketed aggregation), else atomics on the hot slot.
void emit_rank_tail(std::ostringstream& s, const ScanProgram& P) {
  if (P.bkt != nullptr && batched_appends()) {
    // all R reservations first (independent atomics in flight together), then the stores: one
    // atomic round trip per tile instead of R serialised ones (the consume profile showed the
    // warps waiting on each append's return in turn)
    s << "      { uint64_t ab[R]; unsigned apos[R];\n"
      << "#pragma unroll\n      for (int r = 0; r < R; ++r) { ab[r] = 0; apos[r] = 0; if (!(pass & (1u << r))) continue;\n"
      << "        ab[r] = ((sl[r] >> " << kBucketBits << ") << P.bkt_sub_bits) | (threadIdx.x & ((1u << P.bkt_sub_bits) - 1u));\n"
      << "        apos[r] = atomicAdd(P.bkt_fill + ab[r], 1u); }\n"
      << "#pragma unroll\n      for (int r = 0; r < R; ++r) { if (!(pass & (1u << r))) continue;\n"
      << "        uint64_t e = sl[r] & " << (kBucketSlots - 1) << "ULL;\n";
    for (int k = 0; k < P.n_sum; ++k)
      s << "        e |= ((" << V(P.sum_reg[k]) << "[r] - static_cast<uint64_t>(P.bkt_min[" << k << "])) & P.bkt_mask[" << k
        << "]) << P.bkt_shift[" << k << "];\n";
    s << "        if (apos[r] < P.bkt_cap) {\n"
      << "          P.bkt[ab[r] * P.bkt_cap + apos[r]] = e;\n        } else {  // bucket full: the overflow list\n"
      << "          const unsigned o = atomicAdd(P.bkt_ovf_count, 1u);\n"
      << "          if (o < P.bkt_ovf_cap) { P.bkt_ovf[2 * o] = sl[r]; P.bkt_ovf[2 * o + 1] = e; }\n        }\n"
      << "      } }\n";
    return;
  }
  s << "#pragma unroll\n      for (int r = 0; r < R; ++r) { if (!(pass & (1u << r))) continue;\n";
  if (P.bkt != nullptr) {  // append one word to the slot's bucket (k_bucket_emit folds it)
    s << "        const uint64_t b = ((sl[r] >> " << kBucketBits << ") << P.bkt_sub_bits) | (threadIdx.x & ((1u << P.bkt_sub_bits) - 1u));\n"
      << "        const unsigned pos = atomicAdd(P.bkt_fill + b, 1u);\n"
      << "        uint64_t e = sl[r] & " << (kBucketSlots - 1) << "ULL;\n";
    for (int k = 0; k < P.n_sum; ++k)
      s << "        e |= ((" << V(P.sum_reg[k]) << "[r] - static_cast<uint64_t>(P.bkt_min[" << k << "])) & P.bkt_mask[" << k
        << "]) << P.bkt_shift[" << k << "];\n";
    s << "        if (pos < P.bkt_cap) {\n";
    s << "          P.bkt[b * P.bkt_cap + pos] = e;\n        } else {  // bucket full: the overflow list\n"
      << "          const unsigned o = atomicAdd(P.bkt_ovf_count, 1u);\n"
      << "          if (o < P.bkt_ovf_cap) { P.bkt_ovf[2 * o] = sl[r]; P.bkt_ovf[2 * o + 1] = e; }\n        }\n"
      << "        continue;\n";
  }
  s << "        unsigned long long* h = reinterpret_cast<unsigned long long*>(T.hot + sl[r] * " << P.agg.hw << ");\n";
  emit_accumulate(s, P, "        ");
  s << "      }\n";
}

/// Peer-slab shuffle (P.slab, SINK_PROBE at N > 1): the rows owned by other ranks go into the
/// outbox region of their destination in CHUNKS of kSlabChunk words a warp claims with one atomic
/// (per-row reservations on one counter serialised at the L2: SF100 N=2 probe 1.7 -> 6.8 ms; a
/// shared-memory staging buffer with per-flush reservations cost ~320 extra warp instructions per
/// tile, profiles/r2_ncu_probe_fake.txt). The lanes of a warp with the same destination store
/// consecutive words of the warp's current chunk; a chunk left partly filled (a new chunk was
/// claimed, or the kernel ends) is padded with the sentinel word 1 << 63, never a packed row
/// (slab mode requires packed rows of at most 63 bits). Chunk state per (warp, destination) lives
/// in shared memory, updated warp-synchronously. `w` indexes the warp's state row.
/// PSG_SLAB_DIAG (measurement only - results are wrong when set): 1 no outbox stores, 2 remote
/// rows dropped, 8 remote rows screened through the own rank records (the one-GPU lookup
/// footprint) instead of the global bitmap.
/// PSG_TILE_PUT=1: the per-tile outbox placement also at more than two ranks (once per
/// destination) - measured slower at N=4 (probe 1.13 -> 1.32 ms), so the per-row-slot
/// match-based put stays the default there.
bool tile_put_env() {
  static const bool v = [] {
    const char* e = std::getenv("PSG_TILE_PUT");
    return e && e[0] == '1';
  }();
  return v;
}
int slab_diag() {
  static const int v = [] {
    const char* e = std::getenv("PSG_SLAB_DIAG");
    return e ? std::atoi(e) : 0;
  }();
  return v;
}
constexpr int kSlabChunk = 256;

void emit_slab_prologue(std::ostringstream& s, const ScanProgram& P, int nwarps, const std::string& w) {
  s << "  __shared__ unsigned long long s_cbase[" << nwarps << "][" << P.nparts << "];\n"
    << "  __shared__ unsigned s_cfill[" << nwarps << "][" << P.nparts << "];\n"
    // warp-private state rows: each warp initialises its own (no block barrier: the warp-specialised
    // kernel's producer warp has already left)
    << "  for (int i = threadIdx.x & 31; i < " << P.nparts << "; i += 32) { s_cfill[" << w << "][i] = " << kSlabChunk
    << "u; s_cbase[" << w << "][i] = ~0ULL; }\n  __syncwarp();\n"
    // pad the rest of the chunk [from, kSlabChunk) of destination d with sentinels (lanes of `grp`)
    << "  auto slab_pad = [&](unsigned grp, uint32_t d, unsigned long long base, unsigned from) {\n"
    << "    if (base == ~0ULL) return;\n"
    << "    const unsigned me = __popc(grp & ((1u << (threadIdx.x & 31)) - 1u)), n = __popc(grp);\n"
    << "    for (unsigned i = from + me; i < " << kSlabChunk << "u; i += n) if (base + i < P.slab_cap) P.slab_dst[d][base + i] = 1ULL << 63;\n"
    << "  };\n"
    // append one word per lane of `on` lanes; dst per lane
    << "  auto slab_put = [&](bool on, uint32_t d, uint64_t word) {\n"
    << "    const unsigned grp = __match_any_sync(0xffffffffu, on ? d : 0xffffffffu);\n"
    << "    if (on) {\n"
    << "      const int leader = __ffs(grp) - 1; const unsigned cnt = __popc(grp);\n"
    << "      unsigned fill = s_cfill[" << w << "][d]; unsigned long long base = s_cbase[" << w << "][d];\n"
    << "      if (fill + cnt > " << kSlabChunk << "u) {\n"
    << "        slab_pad(grp, d, base, fill);\n"
    << "        if ((threadIdx.x & 31) == leader) base = atomicAdd(P.slab_cnt + d, " << kSlabChunk << "ULL);\n"
    << "        base = __shfl_sync(grp, base, leader); fill = 0;\n      }\n"
    << "      const unsigned long long pos = base + fill + __popc(grp & ((1u << (threadIdx.x & 31)) - 1u));\n"
    << "      if (pos < P.slab_cap" << ((slab_diag() & 1) ? " && pos == ~0ULL" : "") << ") P.slab_dst[d][pos] = word;\n"
    << "      __syncwarp(grp);\n"
    << "      if ((threadIdx.x & 31) == leader) { s_cfill[" << w << "][d] = fill + cnt; s_cbase[" << w << "][d] = base; }\n"
    << "    }\n    __syncwarp();\n  };\n"
    ;
  // two ranks: one destination, chunk state in (warp-uniform) registers, ballot instead of match
  if (P.nparts == 2)
    s << "  unsigned c2fill = " << kSlabChunk << "u; unsigned long long c2base = ~0ULL;\n"
    << "  auto slab_put2 = [&](bool on, uint64_t word) {\n"
    << "    const unsigned b = __ballot_sync(0xffffffffu, on);\n    if (!b) return;\n"
    << "    const unsigned cnt = __popc(b);\n"
    << "    if (c2fill + cnt > " << kSlabChunk << "u) {\n"
    << "      slab_pad(0xffffffffu, " << 1 - P.self_rank << "u, c2base, c2fill);\n"
    << "      unsigned long long nb = 0;\n"
    << "      if ((threadIdx.x & 31) == 0) nb = atomicAdd(P.slab_cnt + " << 1 - P.self_rank << ", " << kSlabChunk << "ULL);\n"
    << "      c2base = __shfl_sync(0xffffffffu, nb, 0); c2fill = 0;\n    }\n"
    << "    const unsigned long long pos = c2base + c2fill + __popc(b & ((1u << (threadIdx.x & 31)) - 1u));\n"
    << "    if (on && pos < P.slab_cap" << ((slab_diag() & 1) ? " && pos == ~0ULL" : "") << ") P.slab_dst[" << 1 - P.self_rank << "][pos] = word;\n"
    << "    c2fill += cnt;\n  };\n";
  // kernel end: pad every partly filled chunk of this warp
  s << "  auto slab_finish = [&]() {\n    __syncwarp();\n";
  if (P.nparts == 2) s << "    slab_pad(0xffffffffu, " << 1 - P.self_rank << "u, c2base, c2fill);\n";
  // (chunks of the match-based put; untouched rows keep base ~0: no-op)
  s << "    for (uint32_t d = 0; d < " << P.nparts << "u; ++d) slab_pad(0xffffffffu, d, s_cbase[" << w << "][d], s_cfill[" << w << "][d]);\n";
  s << "  };\n";
}

/// Default peer-slab probe (PSG_SLAB_V=2: the branchy two-lookup emit_slab_probe2): branch-free -
/// every row issues ONE 16-byte load whose base depends on its owner (own rank records, or the
/// 16-byte chunk of the global bitmap holding its bit), so the warp does not diverge into two
/// lookup paths; two ranks use the ballot-based register-state put.
template <class Late>
void emit_slab_probe3(std::ostringstream& s, const ScanProgram& P, Late late) {
  // (slots and ranks in 32 bits: the engine caps a rank table at 2^32 keys; fewer registers at the
  // 60-register cap of 2 x 544-thread CTAs per SM)
  s << "    { const AggTableDev& T = P.agg; unsigned long long bw[R]; uint32_t bp[R], sl[R], bb[R], dst[R];\n"
    << "      uint32_t own = 0, rem = 0;\n"
    << "      const unsigned long long* gbits = reinterpret_cast<const unsigned long long*>(P.semi_kbits);\n"
    << "#pragma unroll\n      for (int r = 0; r < R; ++r) { const uint64_t key = " << V(P.key_reg) << "[r];\n"
    << "        const uint64_t d = key - static_cast<uint64_t>(T.kmin);\n"
    << "        const bool ok = ((pass >> r) & 1u) && key != kEmptyKey && d < T.krange;\n"
    << "        const uint32_t o = part_of(key, " << P.nparts << "u); dst[r] = o;\n"
    << "        const bool mine = o == " << P.self_rank << "u;\n"
    << "        uint64_t a = 0, b = 0;\n"
    << "        if (ok) ldg_keep_v2u64(mine ? T.krec + 2 * (d >> 6) : gbits + 2 * (d >> 7), pol_keep, a, b);\n"
    << "        bb[r] = static_cast<uint32_t>(d & 63);\n"
    << "        bw[r] = (mine || !((d >> 6) & 1)) ? a : b; bp[r] = mine ? static_cast<uint32_t>(b) : 0u;\n"
    << "        own |= static_cast<uint32_t>(ok && mine) << r; rem |= static_cast<uint32_t>(ok && !mine) << r; }\n"
    << "#pragma unroll\n      for (int r = 0; r < R; ++r) {\n"
    << "        if (!((bw[r] >> bb[r]) & 1ULL)) { own &= ~(1u << r); rem &= ~(1u << r); }\n"
    << "        sl[r] = bp[r] + static_cast<uint32_t>(__popcll(bw[r] & ((1ULL << bb[r]) - 1ULL))); }\n"
    << "      pass = own | rem;\n";
  late();
  if (slab_diag() & 2) s << "      rem = 0;\n";
  s << "#pragma unroll\n      for (int r = 0; r < R; ++r) {\n"
    << "        const bool on = (rem >> r) & 1u;\n";
  if (P.nparts == 2)
    s << "        slab_put2(on, on ? " << out_value(P, 0) << " : 0ULL);\n      }\n";
  else
    s << "        if (__any_sync(0xffffffffu, on)) slab_put(on, dst[r], on ? " << out_value(P, 0) << " : 0ULL);\n      }\n";
  s << "      pass = own;\n";
  emit_rank_tail(s, P);
  s << "    }\n";
}

/// The probe with the peer-slab shuffle: ONE dependent 16-byte lookup per row into the global
/// records {global key-bitmap word, own rank at the word} (the same footprint as the one-GPU rank
/// records). A key absent from the global bitmap drops the row; a key this rank owns gets its slot
/// = own rank + the own keys below it in the word (the set global bits below it whose key hashes
/// to this rank - a handful of multiply-shifts); any other key's row is staged (bit-packed, with
/// its destination) for the slab flush. `late` loads the non-key columns of the survivors.
template <class Late>
void emit_slab_probe1(std::ostringstream& s, const ScanProgram& P, Late late, const std::string& w) {
  s << "    { const AggTableDev& T = P.agg; unsigned long long gw[R]; uint32_t orr[R], sl[R], bb[R], dst[R];\n"
    << "      uint32_t own = 0, rem = 0;\n"
    << "#pragma unroll\n      for (int r = 0; r < R; ++r) { gw[r] = 0; orr[r] = 0; bb[r] = 0; dst[r] = 0; const uint64_t key = "
    << V(P.key_reg) << "[r];\n"
    << "        if ((pass & (1u << r)) && key != kEmptyKey) { const uint64_t d = key - static_cast<uint64_t>(T.kmin);\n"
    << "          if (d < T.krange) { bb[r] = static_cast<uint32_t>(d & 63); dst[r] = part_of(key, static_cast<uint32_t>(P.nparts));\n"
    << "            uint64_t a, b; ldg_keep_v2u64(P.slab_grec + 2 * (d >> 6), pol_keep, a, b); gw[r] = a; orr[r] = static_cast<uint32_t>(b); } } }\n"
    << "#pragma unroll\n      for (int r = 0; r < R; ++r) { sl[r] = 0;\n"
    << "        if (!((gw[r] >> bb[r]) & 1ULL)) continue;\n"
    << "        if (dst[r] != static_cast<uint32_t>(P.self_rank)) { rem |= 1u << r; continue; }\n"
    << "        own |= 1u << r;\n"
    << "        const uint64_t base = " << V(P.key_reg) << "[r] - bb[r];\n"
    << "        unsigned long long m = gw[r] & ((1ULL << bb[r]) - 1ULL); uint32_t c = orr[r];\n"
    << "        while (m) { const int i = __ffsll(static_cast<long long>(m)) - 1; m &= m - 1;\n"
    << "          if (part_of(base + i, static_cast<uint32_t>(P.nparts)) == static_cast<uint32_t>(P.self_rank)) ++c; }\n"
    << "        sl[r] = c; }\n"
    << "      pass = own | rem;\n";
  late();
  if (slab_diag() & 2) s << "      rem = 0;\n";
  s << "#pragma unroll\n      for (int r = 0; r < R; ++r) {\n"
    << "        const bool on = (rem >> r) & 1u;\n"
    << "        if (__any_sync(0xffffffffu, on)) slab_put(on, dst[r], on ? " << out_value(P, 0) << " : 0ULL);\n      }\n"
    << "      pass = own;\n";
  emit_rank_tail(s, P);
  s << "    }\n";
}

/// The probe with the peer-slab shuffle: ONE dependent lookup per row, chosen by its owner -
/// a row this rank owns reads its 16-byte rank record (membership + slot, as at one GPU), any
/// other row the word of the global key bitmap (the exact semi-join screen). `late` then loads
/// the non-key columns of the survivors; remote survivors are staged (bit-packed, with their
/// destination) for the slab flush, owned survivors accumulate into their slots.
template <class Late>
void emit_slab_probe2(std::ostringstream& s, const ScanProgram& P, Late late, const std::string& w) {
  s << "    { const AggTableDev& T = P.agg; unsigned long long bw[R]; uint64_t bp[R], sl[R]; uint32_t bb[R], dst[R];\n"
    << "      uint32_t own = 0, rem = 0;\n"
    << "#pragma unroll\n      for (int r = 0; r < R; ++r) { bw[r] = 0; bp[r] = 0; bb[r] = 0; dst[r] = 0; const uint64_t key = "
    << V(P.key_reg) << "[r];\n"
    << "        if ((pass & (1u << r)) && key != kEmptyKey) { const uint64_t d = key - static_cast<uint64_t>(T.kmin);\n"
    << "          if (d < T.krange) { const uint32_t o = part_of(key, " << P.nparts << "u); dst[r] = o;\n"
    << "            if (o == " << P.self_rank << "u) { own |= 1u << r; bb[r] = static_cast<uint32_t>(d & 63);\n"
    << "              uint64_t a, b; ldg_keep_v2u64(T.krec + 2 * (d >> 6), pol_keep, a, b); bw[r] = a; bp[r] = b; }\n"
    << "            else { rem |= 1u << r; " << ((slab_diag() & 8) ? "bb[r] = static_cast<uint32_t>(d & 63); uint64_t a, b; ldg_keep_v2u64(T.krec + 2 * (d >> 6), pol_keep, a, b); bw[r] = ~0ULL; bp[r] = a + b;" : "bb[r] = static_cast<uint32_t>(d & 31); bw[r] = ldg_keep_u32(P.semi_kbits + (d >> 5), pol_keep);") << " } } } }\n"
    << "#pragma unroll\n      for (int r = 0; r < R; ++r) { sl[r] = 0;\n"
    << "        if (!((bw[r] >> bb[r]) & 1ULL)) { own &= ~(1u << r); rem &= ~(1u << r); }\n"
    << "        else if ((own >> r) & 1u) sl[r] = bp[r] + static_cast<uint64_t>(__popcll(bw[r] & ((1ULL << bb[r]) - 1ULL))); }\n"
    << "      pass = own | rem;\n";
  late();
  if (slab_diag() & 2) s << "      rem = 0;\n";
  s << "#pragma unroll\n      for (int r = 0; r < R; ++r) {\n"
    << "        const bool on = (rem >> r) & 1u;\n"
    << "        if (__any_sync(0xffffffffu, on)) slab_put(on, dst[r], on ? " << out_value(P, 0) << " : 0ULL);\n      }\n"
    << "      pass = own;\n";
  emit_rank_tail(s, P);
  s << "    }\n";
}

/// PSG_SLAB_GREC=1: the one-lookup variant over the global records (emit_slab_probe1); default the
/// two-lookup variant (emit_slab_probe2: own rank records / global bitmap by owner).
bool slab_grec_env() {
  static const bool v = [] {
    const char* e = std::getenv("PSG_SLAB_GREC");
    return e && e[0] == '1';
  }();
  return v;
}
/// Screen-first peer-slab probe (default; PSG_SLAB_V=3: the one-lookup branch-free variant; SF100
/// N=2 A/B: probe 2.34 -> 2.04 ms, query 3.66 -> 3.36 ms): every
/// predicate-passing row tests its bit in the 4-byte word of the GLOBAL key bitmap (19 MB at SF100
/// - half the rank records' footprint, so more of the 300 M lookups hit L2); only the ~10% that
/// survive compute their owner, and the owned ones read their rank record (slot) together with
/// the late columns - the extra lookup overlaps the HBM gathers.
template <class Late>
void emit_slab_probe4(std::ostringstream& s, const ScanProgram& P, Late late, const std::string& w) {
  s << "    { const AggTableDev& T = P.agg; uint32_t gw[R], bb[R], kr[R], sl[R], dst[R]; unsigned long long kw[R];\n"
    << "      uint32_t sel = 0, own = 0, rem = 0;\n"
    << "#pragma unroll\n      for (int r = 0; r < R; ++r) { const uint64_t key = " << V(P.key_reg) << "[r];\n"
    << "        const uint64_t d = key - static_cast<uint64_t>(T.kmin);\n"
    << "        const bool ok = ((pass >> r) & 1u) && key != kEmptyKey && d < T.krange;\n"
    << "        bb[r] = static_cast<uint32_t>(d & 31); gw[r] = ok ? ldg_keep_u32(P.semi_kbits + (d >> 5), pol_keep) : 0u; }\n"
    << "#pragma unroll\n      for (int r = 0; r < R; ++r) if ((gw[r] >> bb[r]) & 1u) sel |= 1u << r;\n"
    << "#pragma unroll\n      for (int r = 0; r < R; ++r) { dst[r] = 0; kw[r] = 0; kr[r] = 0;\n"
    << "        if ((sel >> r) & 1u) { const uint64_t key = " << V(P.key_reg) << "[r];\n"
    << "          const uint32_t o = part_of(key, " << P.nparts << "u); dst[r] = o;\n"
    << "          if (o == " << P.self_rank << "u) { own |= 1u << r; const uint64_t d = key - static_cast<uint64_t>(T.kmin);\n"
    << "            uint64_t a, b; ldg_keep_v2u64(T.krec + 2 * (d >> 6), pol_keep, a, b); kw[r] = a; kr[r] = static_cast<uint32_t>(b); }\n"
    << "          else rem |= 1u << r; } }\n"
    << "      pass = sel;\n";
  late();
  s << "#pragma unroll\n      for (int r = 0; r < R; ++r) { const uint32_t d6 = static_cast<uint32_t>((" << V(P.key_reg)
    << "[r] - static_cast<uint64_t>(T.kmin)) & 63);\n"
    << "        sl[r] = kr[r] + static_cast<uint32_t>(__popcll(kw[r] & ((1ULL << d6) - 1ULL))); }\n";
  if (slab_diag() & 2) s << "      rem = 0;\n";
  if (P.nparts == 2) {
    // two ranks: one destination, so the tile's remote rows are placed with ONE chunk check - a
    // ballot per row slot, positions from the running count; rows past the current chunk's room
    // go to a freshly claimed one (at most one per tile: a tile has R x 32 < kSlabChunk rows)
    s << "      { unsigned bl[R], tot = 0; const uint32_t lt = (1u << (threadIdx.x & 31)) - 1u;\n"
      << "#pragma unroll\n        for (int r = 0; r < R; ++r) { bl[r] = __ballot_sync(0xffffffffu, (rem >> r) & 1u); tot += __popc(bl[r]); }\n"
      << "        if (tot) {\n"
      << "          const unsigned room = c2base == ~0ULL ? 0u : " << kSlabChunk << "u - c2fill;\n"
      << "          unsigned long long nb = c2base;\n"
      << "          if (tot > room) {\n"
      << "            if ((threadIdx.x & 31) == 0) nb = atomicAdd(P.slab_cnt + " << 1 - P.self_rank << ", " << kSlabChunk << "ULL);\n"
      << "            nb = __shfl_sync(0xffffffffu, nb, 0);\n          }\n"
      << "          unsigned at = 0;\n"
      << "#pragma unroll\n          for (int r = 0; r < R; ++r) {\n"
      << "            if ((rem >> r) & 1u) { const unsigned k = at + __popc(bl[r] & lt);\n"
      << "              const unsigned long long pos = k < room ? c2base + c2fill + k : nb + (k - room);\n"
      << "              if (pos < P.slab_cap" << ((slab_diag() & 1) ? " && pos == ~0ULL" : "") << ") P.slab_dst[" << 1 - P.self_rank
      << "][pos] = " << out_value(P, 0) << "; }\n"
      << "            at += __popc(bl[r]); }\n"
      << "          if (tot > room) { c2base = nb; c2fill = tot - room; } else { c2fill += tot; }\n"
      << "        }\n      }\n";
  } else if (tile_put_env()) {
    // more ranks: the same per-tile placement once per destination (literal loop over the ranks,
    // chunk state of the warp in shared memory)
    s << "      { const uint32_t lt = (1u << (threadIdx.x & 31)) - 1u;\n";
    for (int d = 0; d < P.nparts; ++d) {
      if (d == P.self_rank) continue;
      s << "      { unsigned bl[R], tot = 0;\n"
        << "#pragma unroll\n        for (int r = 0; r < R; ++r) { bl[r] = __ballot_sync(0xffffffffu, ((rem >> r) & 1u) && dst[r] == " << d
        << "u); tot += __popc(bl[r]); }\n"
        << "        if (tot) {\n"
        << "          unsigned cf = s_cfill[" << w << "][" << d << "]; unsigned long long cb = s_cbase[" << w << "][" << d << "];\n"
        << "          const unsigned room = cb == ~0ULL ? 0u : " << kSlabChunk << "u - cf;\n"
        << "          unsigned long long nb = cb;\n"
        << "          if (tot > room) {\n"
        << "            if ((threadIdx.x & 31) == 0) nb = atomicAdd(P.slab_cnt + " << d << ", " << kSlabChunk << "ULL);\n"
        << "            nb = __shfl_sync(0xffffffffu, nb, 0);\n          }\n"
        << "          unsigned at = 0;\n"
        << "#pragma unroll\n          for (int r = 0; r < R; ++r) {\n"
        << "            if ((bl[r] >> (threadIdx.x & 31)) & 1u) { const unsigned k = at + __popc(bl[r] & lt);\n"
        << "              const unsigned long long pos = k < room ? cb + cf + k : nb + (k - room);\n"
        << "              if (pos < P.slab_cap) P.slab_dst[" << d << "][pos] = " << out_value(P, 0) << "; }\n"
        << "            at += __popc(bl[r]); }\n"
        << "          __syncwarp();\n"
        << "          if ((threadIdx.x & 31) == 0) { if (tot > room) { s_cbase[" << w << "][" << d << "] = nb; s_cfill[" << w << "][" << d
        << "] = tot - room; } else { s_cfill[" << w << "][" << d << "] = cf + tot; } }\n"
        << "          __syncwarp();\n        }\n      }\n";
    }
    s << "      }\n";
  } else {
    s << "#pragma unroll\n      for (int r = 0; r < R; ++r) {\n"
      << "        const bool on = (rem >> r) & 1u;\n"
      << "        if (__any_sync(0xffffffffu, on)) slab_put(on, dst[r], on ? " << out_value(P, 0) << " : 0ULL);\n      }\n";
  }
  s << "      pass = own;\n";
  emit_rank_tail(s, P);
  s << "    }\n";
}

int slab_variant() {
  static const int v = [] {
    const char* e = std::getenv("PSG_SLAB_V");
    return e ? std::atoi(e) : 4;
  }();
  return v;
}
template <class Late>
void emit_slab_probe(std::ostringstream& s, const ScanProgram& P, Late late, const std::string& w) {
  if (P.slab_grec != nullptr && slab_grec_env())
    emit_slab_probe1(s, P, late, w);
  else if (slab_variant() == 2)
    emit_slab_probe2(s, P, late, w);
  else if (slab_variant() == 3)
    emit_slab_probe3(s, P, late);
  else
    emit_slab_probe4(s, P, late, w);
}

/// SINK_KEYBITS: every surviving row sets its key's bit. With kb_flag a duplicate (bit already
/// set) or out-of-range key raises the flag (atomics with a return value: the warp waits on them);
/// without it the bits are set by reductions (no return, nothing to wait for) and the engine
/// detects duplicates / out-of-range keys as fewer set bits than rows (kb_count).
void emit_keybits(std::ostringstream& s, const ScanProgram& P) {
  s << "    { unsigned nset = 0;\n#pragma unroll\n      for (int r = 0; r < R; ++r) { if (!(pass & (1u << r))) continue;\n"
    << "        const uint64_t d = " << V(P.key_reg) << "[r] - static_cast<uint64_t>(P.kb_min);\n"
    << "        ++nset;\n";
  if (P.kb_flag != nullptr)
    s << "        if (d >= P.kb_range) { atomicOr(P.kb_flag, 2u); continue; }\n"
      << "        const uint32_t bit = 1u << (d & 31);\n"
      << "        if (atomicOr(P.kb_bits + (d >> 5), bit) & bit) atomicOr(P.kb_flag, 1u); }\n";
  else
    s << "        if (d < P.kb_range) atomicOr(P.kb_bits + (d >> 5), 1u << (d & 31)); }\n";
  s << "      kb_rows += nset;\n    }\n";
}

/// Predicate atoms: clear a row's pass bit when an atom fails.
void emit_atoms(std::ostringstream& s, const ScanProgram& P) {
  for (int a = 0; a < P.n_atoms; ++a) {
    const AtomDesc& at = P.atoms[a];
    if (at.is_float) {
      s << "    { const double lit = __longlong_as_double(static_cast<long long>(P.atoms[" << a << "].lit));\n"
        << "#pragma unroll\n      for (int r = 0; r < R; ++r) if (!(__longlong_as_double(static_cast<long long>(" << V(at.reg)
        << "[r])) " << op_str(at.op) << " lit)) pass &= ~(1u << r);\n    }\n";
    } else {
      s << "    { const long long lit = static_cast<long long>(P.atoms[" << a << "].lit);\n"
        << "#pragma unroll\n      for (int r = 0; r < R; ++r) if (!(static_cast<long long>(" << V(at.reg) << "[r]) "
        << op_str(at.op) << " lit)) pass &= ~(1u << r);\n    }\n";
    }
  }
}

/// Unique-key local joins of the chain (two-stage probe: home-slot loads for all rows first).
void emit_joins(std::ostringstream& s, const ScanProgram& P) {
  for (int j = 0; j < P.n_joins; ++j) {
    const JoinDesc& jd = P.joins[j];
    if (jd.t.bitmap != nullptr) {  // dense unique keys, no payload: membership bitmap (L2-resident)
      s << "    { const LocalTableDev& T = P.joins[" << j << "].t;\n"
        << "#pragma unroll\n      for (int r = 0; r < R; ++r) if ((pass & (1u << r)) && !local_bitmap_has(T, " << V(jd.key_reg)
        << "[r])) pass &= ~(1u << r);\n    }\n";
      continue;
    }
    s << "    { const LocalTableDev& T = P.joins[" << j << "].t;\n      uint64_t sl[R], k0[R];\n"
      << "#pragma unroll\n      for (int r = 0; r < R; ++r) { sl[r] = ~0ULL; k0[r] = 0; if (pass & (1u << r)) {\n"
      << "        const uint64_t key = " << V(jd.key_reg) << "[r];\n"
      << "        if (key == kEmptyKey) { if (T.cnt[T.mask + 1] == 0) pass &= ~(1u << r); else { sl[r] = T.mask + 1; k0[r] = key; } }\n"
      << "        else { sl[r] = slot_of(key, T.shift); k0[r] = T.keys[sl[r]]; } } }\n"
      << "#pragma unroll\n      for (int r = 0; r < R; ++r) { if (!(pass & (1u << r))) continue;\n"
      << "        const uint64_t key = " << V(jd.key_reg) << "[r]; uint64_t sx = sl[r], kk = k0[r];\n"
      << "        if (sx != T.mask + 1) { while (kk != key && kk != kEmptyKey) { sx = (sx + 1) & T.mask; kk = T.keys[sx]; }\n"
      << "          if (kk != key) { pass &= ~(1u << r); continue; } }\n";
    if (jd.t.npayload > 0) {
      s << "        const uint32_t st = T.start[sx];\n";
      for (int p = 0; p < jd.t.npayload; ++p)
        s << "        " << V(jd.payload_reg[p]) << "[r] = T.payload[" << p << "][st];\n";
    }
    s << "      }\n    }\n";
  }
}

/// Semi-join screen of a partitioning scan (MATERIALIZE with nparts > 1): drop rows whose key is
/// certainly absent on its owner rank - exact global key bitmap, or the owner's Bloom filter.
/// Two stages: all R filter words in flight before any test.
void emit_semi_screen(std::ostringstream& s, const ScanProgram& P) {
  if (P.semi_kbits != nullptr) {  // exact global key bitmap
    // two stages, like the Bloom screen: all R bitmap words in flight before any test
    s << "    { uint32_t bw[R], bb[R];\n"
      << "#pragma unroll\n      for (int r = 0; r < R; ++r) { bw[r] = 1u; bb[r] = 0u; const uint64_t key = "
      << V(P.semi_key_reg) << "[r];\n"
      << "        if ((pass & (1u << r)) && key != kEmptyKey) { const uint64_t d = key - static_cast<uint64_t>(P.semi_kmin);\n"
      << "          bw[r] = 0u; if (d < P.semi_krange) { bb[r] = static_cast<uint32_t>(d & 31); "
         "bw[r] = ldg_keep_u32(P.semi_kbits + (d >> 5), pol_keep); } } }\n"
      << "#pragma unroll\n      for (int r = 0; r < R; ++r) if (!((bw[r] >> bb[r]) & 1u)) pass &= ~(1u << r);\n    }\n";
  } else if (P.semi_bloom != nullptr) {
    s << "    { uint32_t bw[R], bm[R];\n"
      << "#pragma unroll\n      for (int r = 0; r < R; ++r) { bw[r] = bm[r] = 0; const uint64_t key = " << V(P.semi_key_reg)
      << "[r];\n        if ((pass & (1u << r)) && key != kEmptyKey) { const uint64_t h2 = key * kBloomMul;\n"
      << "          const uint32_t d = part_of(key, static_cast<uint32_t>(P.nparts));\n"
      << "          bm[r] = bloom_bits(h2, P.semi_shift); bw[r] = ldg_keep_u32(P.semi_bloom + d * P.semi_words + (h2 >> P.semi_shift), pol_keep); } }\n"
      << "#pragma unroll\n      for (int r = 0; r < R; ++r) if ((pass & (1u << r)) && (bw[r] & bm[r]) != bm[r]) pass &= ~(1u << r);\n    }\n";
  }
}

/// Warp-specialised probe for the one-GPU rank-indexed table (PSG_TMA=0: off). Shape knobs:
/// PSG_TMA_NG consumer groups of 8 warps (default 2), PSG_TMA_NS ring stages (4), PSG_TMA_CTAS
/// CTAs per SM (2).
struct StagedShape {
  int groups, stages, ctas, rows;  // rows: per consumer lane per tile (4 or 8); 1024 / (32 rows) warps per group
  int warps() const { return 1024 / (32 * rows); }
};
StagedShape staged_shape() {
  static const StagedShape sh = [] {
    auto env = [](const char* n, int d) {
      const char* e = std::getenv(n);
      return e ? std::max(1, std::atoi(e)) : d;
    };
    const int r = env("PSG_TMA_R", 4) >= 8 ? 8 : 4;
    return StagedShape{env("PSG_TMA_NG", 2), env("PSG_TMA_NS", 4), env("PSG_TMA_CTAS", 2), r};
  }();
  return sh;
}
bool staged_probe(const ScanProgram& P) {
  static const bool on = [] {
    const char* e = std::getenv("PSG_TMA");
    return !(e && e[0] == '0');
  }();
  if (!on || !P.staged_ok || P.remote || P.unpack_n != 0 || P.n_early < 1 || P.n_early > 4 || P.n_in > kMaxIn) return false;
  if (P.sink == SINK_PROBE) return P.agg.krec != nullptr;
  // the key-bitmap build (orders: date + customer key early, the order key late): opt-in
  // (PSG_TMA_KB=1) - measured slower than the register kernel (SF100 N=1 orders scan 0.91 vs
  // 0.75 ms: its chain date -> customer bitmap -> order key -> bit is short per row)
  static const bool kb_on = [] {
    const char* e = std::getenv("PSG_TMA_KB");
    return e && e[0] == '1';
  }();
  if (P.sink == SINK_KEYBITS) return kb_on;
  // unordered warp-staged compaction (+ partition histogram, semi-join screen, packed rows):
  // opt-in (PSG_TMA_MAT=1) - the SF100 orders scan measured slower staged (0.97 vs 0.73 ms: three
  // early columns leave room for one CTA per SM)
  static const bool mat_on = [] {
    const char* e = std::getenv("PSG_TMA_MAT");
    return e && e[0] == '1';
  }();
  return mat_on && P.sink == SINK_MATERIALIZE && P.tile_offsets == nullptr && P.n_out >= 1 && P.n_out <= 4 &&
         !P.self_probe;
}

/// Rows per thread per tile (R) of the kernel: R x 32 rows per warp, 1024 / (32 R) warps per
/// block (a tile is always 1024 rows).
int jit_rows(const ScanProgram& P) {
  // PSG_JIT_R: 4 | 8 (every program) | p (probe sinks at 8: default) | pm (probe + materialise).
  // The probe programs are latency-bound on their chain of dependent loads (predicate, key
  // bitmap, home slot, sums): 8 rows per thread at 64 registers (4 warps x 8 CTAs per SM) keep
  // 8192 rows in flight per SM vs 6144 at R = 4, 40 registers, 6 x 8 warps. Measured SF100:
  // N=1 query 7.69/7.64 -> 7.49/7.44 ms (probe kernel 4.37/4.41 -> 4.23/4.20), N=2 6.00 -> 5.95;
  // the partitioning materialise programs are slower at R = 8 (N=2 probe-side scan 2.15 -> 2.68).
  static const std::string env = [] {
    const char* e = std::getenv("PSG_JIT_R");
    return std::string(e ? e : "p");
  }();
  if (env == "8") return 8;
  const bool probe = P.sink == SINK_PROBE || P.sink == SINK_PROBE_GLOBAL;
  if (env == "p") return probe ? 8 : 4;
  if (env == "pm") return probe || P.sink == SINK_MATERIALIZE ? 8 : 4;
  if (env == "pk") return probe || P.sink == SINK_KEYBITS ? 8 : 4;
  return 4;
}
int jit_block(const ScanProgram& P) { return 1024 / jit_rows(P); }

/// CTAs per SM the kernel is compiled for (register cap 65536 / (256 x this)). PSG_JIT_MINB
/// overrides it (measurement knob).
int min_blocks(const ScanProgram& P) {
  static const int env = [] {
    const char* e = std::getenv("PSG_JIT_MINB");
    return e ? std::atoi(e) : 0;
  }();
  if (env > 0) return env;
  // the key-bitmap build (date -> customer bitmap -> key -> bit): 8 CTAs/SM at 32 registers, no
  // spills (SF100 N=1 query 4.44 -> 4.38 ms with every register program at 8)
  if (P.sink == SINK_KEYBITS) return 8;
  // 6 x 256 threads: 40 registers. At 8 (32 registers) the probe/build programs spill 16-64 B
  // per thread, and the local-memory stores go through to L2 (8 GB per SF100 probe launch in the
  // ncu capture); A/B at N=1 SF100: probe kernel 4.47/4.52 -> 4.42/4.35 ms, query 7.90/7.95 ->
  // 7.74/7.67 ms; 4 CTAs/SM (52 registers, no spills) is slower (5.30 ms).
  return jit_rows(P) == 8 ? 8 : 6;
}

std::string jit_source_staged(const ScanProgram& P);
bool staged_probe(const ScanProgram& P);

std::string jit_source(const ScanProgram& P) {
  if (staged_probe(P)) return jit_source_staged(P);
  std::ostringstream s;
  const int nin = P.n_in, nregs = std::max(1, P.n_regs);
  const bool mat = P.sink == SINK_MATERIALIZE || P.sink == SINK_COUNT;
  const bool probe = P.sink == SINK_PROBE || P.sink == SINK_PROBE_GLOBAL;
  const bool part = P.sink == SINK_MATERIALIZE && P.nparts > 1;
  const bool glob = P.sink == SINK_PROBE_GLOBAL || P.sink == SINK_AGG_SCAN;
  const int nglob = glob ? 1 + P.n_sum + (P.sink == SINK_PROBE_GLOBAL ? P.agg.nbs : 0) : 0;
  // Unordered compaction (pipeline-internal materialisation): each warp stages its surviving rows
  // in shared memory and flushes 128 rows at a time with one global atomic — no block barrier.
  // The order-preserving variant (tile_offsets, SINK_COUNT: the filter op) keeps the block scan.
  const bool wstage = P.sink == SINK_MATERIALIZE && P.tile_offsets == nullptr && P.n_out >= 1 && P.n_out <= 4;
  const bool bscan = mat && !wstage;
  // Block tiles of 1024 rows; warp w owns rows [128w, 128w+128) of the tile, lane-contiguous per
  // r (each warp load = 256 contiguous bytes), so row order inside a tile is (warp, r, lane).
  // Tile descriptors are fetched per warp into registers (lane c holds column c's pointer) and
  // the next tile's descriptor is prefetched while the current one computes: no block barrier
  // except the compaction prefix of the materialising sinks.
  const int RR = jit_rows(P), NT = jit_block(P), NW = NT / 32;
  s << "using namespace psg;\n#define R " << RR << "\n"
    << "extern \"C\" __global__ void __launch_bounds__(" << NT << ", " << min_blocks(P)
    << ") psg_jit_scan(const __grid_constant__ ScanProgram P, "
       "const Segment* __restrict__ segs, const uint32_t* __restrict__ tile_seg, uint64_t ntiles) {\n";
  if (bscan) s << "  __shared__ uint32_t s_wcnt[" << NW << "][R], s_woff[" << NW << "][R];\n  __shared__ unsigned long long s_base;\n";
  if (wstage) s << "  __shared__ uint64_t s_stg[" << NW << "][" << P.n_out << "][128];\n";
  if (part) s << "  __shared__ unsigned long long s_part[" << kMaxParts << "];\n";
  if (glob) s << "  __shared__ unsigned long long s_gacc[" << nglob << "];\n";
  s << "  const int tid = threadIdx.x;\n  const int lane = tid & 31, warp = tid >> 5;\n  const int wrow = warp * (R * 32) + lane;\n"
    << "  const uint64_t pol_keep = l2_evict_last(); (void)pol_keep; (void)wrow;\n";
  if (P.slab) emit_slab_prologue(s, P, NW, "warp");
  // SINK_KEYBITS row count: per lane, one atomic per warp at the end (a per-tile atomic on one
  // counter serialises at the L2)
  if (P.sink == SINK_KEYBITS) s << "  unsigned long long kb_rows = 0;\n";
  if (part) s << "  for (int i = tid; i < " << kMaxParts << "; i += " << NT << ") s_part[i] = 0;\n";
  if (glob) {
    s << "  for (int i = tid; i < " << nglob << "; i += " << NT << ") s_gacc[i] = 0;\n";
    for (int i = 0; i < nglob; ++i)
      s << "  " << (P.global_float[i] ? "double" : "unsigned long long") << " g" << i << " = 0;\n";
  }
  if (part || glob) s << "  __syncthreads();\n";
  s << "  auto fetch = [&](uint64_t t, const uint64_t*& col, uint64_t& r0, int& rows) {\n"
    << "    const Segment* sg = segs + __ldg(tile_seg + t);\n"
    << "    col = lane < " << nin << " ? sg->col[lane] : nullptr;\n"
    << "    r0 = (t - sg->tile_begin) * 1024ULL;\n"
    << "    rows = static_cast<int>(min(1024ULL, sg->rows - r0));\n  };\n";
  if (wstage) {
    s << "  int fill = 0;\n  auto flush = [&]() {\n    __syncwarp();\n    if (fill == 0) return;\n"
      << "    unsigned long long base = 0;\n    if (lane == 0) base = atomicAdd(P.out_count, static_cast<unsigned long long>(fill));\n"
      << "    base = __shfl_sync(0xffffffffu, base, 0);\n"
      << "    for (int i = lane; i < fill; i += 32) { if (base + i >= P.out_cap) continue;\n";
    for (int o = 0; o < P.n_out; ++o) s << "      P.out_col[" << o << "][base + i] = s_stg[warp][" << o << "][i];\n";
    s << "    }\n    fill = 0;\n    __syncwarp();\n  };\n";
  }
  // Contiguous tile ranges per CTA for the warp-staged compaction (non-partitioning programs): a
  // warp's 128 staged survivors then come from adjacent tiles, so the materialised rows stay
  // nearly in scan (key) order instead of runs from tiles a grid apart, and a later scatter by
  // key (the rank table's cold pass) writes longer runs. SF100 N=1 A/B: cold pass 300 -> 250 us,
  // orders scan 743 -> 726 us, query 6.36 -> 6.21 ms (3 pairs). PSG_CONTIG_TILES=0: strided tiles.
  static const bool contig_env = [] {
    const char* e = std::getenv("PSG_CONTIG_TILES");
    return !(e && e[0] == '0');
  }();
  if (wstage && !part && contig_env) {
    s << "  const uint64_t per_cta = (ntiles + gridDim.x - 1) / gridDim.x;\n"
      << "  const uint64_t t_beg = blockIdx.x * per_cta;\n"
      << "  const uint64_t t_end = t_beg + per_cta < ntiles ? t_beg + per_cta : ntiles;\n"
      << "  const uint64_t* cur_col = nullptr; uint64_t cur_r0 = 0; int cur_rows = 0;\n"
      << "  if (t_beg < t_end) fetch(t_beg, cur_col, cur_r0, cur_rows);\n"
      << "  for (uint64_t tile = t_beg; tile < t_end; ++tile) {\n"
      << "    const uint64_t next = tile + 1 < t_end ? tile + 1 : ntiles;\n";
  } else {
    s << "  const uint64_t* cur_col = nullptr; uint64_t cur_r0 = 0; int cur_rows = 0;\n"
      << "  if (blockIdx.x < ntiles) fetch(blockIdx.x, cur_col, cur_r0, cur_rows);\n"
      << "  for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {\n"
      << "    const uint64_t next = tile + gridDim.x;\n";
  }
  s
    << "    const uint64_t* pf_col = nullptr; uint64_t pf_r0 = 0; int pf_rows = 0;\n"
    << "    if (next < ntiles) fetch(next, pf_col, pf_r0, pf_rows);\n"
    << "    const uint64_t row0 = cur_r0;\n    const int nrows = cur_rows - warp * (R * 32);\n"
    << "    uint32_t pass = 0;\n#pragma unroll\n    for (int r = 0; r < R; ++r) if (r * 32 + lane < nrows) pass |= 1u << r;\n";
  for (int r = 0; r < nregs; ++r) s << "    uint64_t " << V(r) << "[R] = {};\n";
  // Phase A: predicate columns + atoms. The early (key) columns are loaded in the same phase, for
  // every valid row: a selective-enough predicate still touches nearly every 32-byte sector of
  // them, and their loads then overlap the predicate loads instead of waiting on the filter
  // (one DRAM round trip fewer on each tile's dependent chain). Measured: SF100 probe kernel
  // 4.36/4.40 -> 4.35/4.31 ms at N=1, neutral at N=2 - the chain's other four round trips (key
  // bitmap, home slot, sums, and the shipdate itself) dominate. PSG_EARLY_KEYS=0: after the filter.
  static const bool early_keys = [] {
    const char* e = std::getenv("PSG_EARLY_KEYS");
    return !(e && e[0] == '0');
  }();
  const bool keys_first = early_keys && P.n_pred > 0 && P.n_early > P.n_pred;
  emit_loads(s, 0, keys_first ? P.n_early : P.n_pred);
  emit_atoms(s, P);
  // Phase B: early columns
  if (!keys_first) emit_loads(s, P.n_pred, P.n_early);
  for (int k = 0; k < P.unpack_n; ++k)  // bit-packed shuffle rows: register 0 -> 1..unpack_n
    s << "#pragma unroll\n    for (int r = 0; r < R; ++r) " << V(1 + k) << "[r] = static_cast<uint64_t>(P.pack_min[" << k
      << "]) + ((" << V(0) << "[r] >> P.pack_shift[" << k << "]) & P.pack_mask[" << k << "]);\n";
  // Phase C: unique-key local joins
  emit_joins(s, P);
  if (P.remote && P.sink == SINK_PROBE) {
    emit_remote_probe(s, P);
  } else if (P.remote && P.sink == SINK_BUILD) {
    emit_loads(s, P.n_early, P.n_in);
    emit_remote_build(s, P);
  } else if (probe && P.agg.krec != nullptr && P.sink == SINK_PROBE && P.slab) {
    emit_slab_probe(s, P, [&] { emit_loads(s, P.n_early, P.n_in); }, "warp");
  } else if (probe && P.agg.krank != nullptr && P.sink == SINK_PROBE) {
    emit_rank_probe(s, P, [&] { emit_loads(s, P.n_early, P.n_in); });
  } else if (probe) {
    const bool bloom = P.agg.bloom != nullptr && P.agg.kbits == nullptr;
    if (P.agg.kbits != nullptr)  // exact membership of dense build keys; all R words in flight first
      s << "    { const AggTableDev& T = P.agg; uint32_t bw[R], bb[R];\n"
        << "#pragma unroll\n      for (int r = 0; r < R; ++r) { bw[r] = 1u; bb[r] = 0u; const uint64_t key = " << V(P.key_reg)
        << "[r];\n        if ((pass & (1u << r)) && key != kEmptyKey) { const uint64_t d = key - static_cast<uint64_t>(T.kmin);\n"
        << "          bw[r] = 0u; if (d < T.krange) { bb[r] = static_cast<uint32_t>(d & 31); "
           "bw[r] = ldg_keep_u32(T.kbits + (d >> 5), pol_keep); } } }\n"
        << "#pragma unroll\n      for (int r = 0; r < R; ++r) if (!((bw[r] >> bb[r]) & 1u)) pass &= ~(1u << r);\n    }\n";
    s << "    { const AggTableDev& T = P.agg;\n      uint64_t sl[R], k0[R];\n";
    if (bloom) {
      s << "      uint32_t bw[R], bm[R];\n"
        << "#pragma unroll\n      for (int r = 0; r < R; ++r) { bw[r] = 0; bm[r] = 0; if ((pass & (1u << r)) && " << V(P.key_reg)
        << "[r] != kEmptyKey) {\n        const uint64_t h2 = " << V(P.key_reg) << "[r] * kBloomMul;\n"
        << "        bm[r] = bloom_bits(h2, T.bloom_shift); bw[r] = ldg_keep_u32(T.bloom + (h2 >> T.bloom_shift), pol_keep); } }\n"
        << "#pragma unroll\n      for (int r = 0; r < R; ++r) if ((pass & (1u << r)) && " << V(P.key_reg)
        << "[r] != kEmptyKey && (bw[r] & bm[r]) != bm[r]) pass &= ~(1u << r);\n";
    }
    s << "#pragma unroll\n      for (int r = 0; r < R; ++r) { sl[r] = ~0ULL; k0[r] = 0; if (pass & (1u << r)) {\n"
      << "        const uint64_t key = " << V(P.key_reg) << "[r];\n"
      << "        if (key == kEmptyKey) { if (T.cold[(T.mask + 1) * T.cw] == 0) pass &= ~(1u << r); else sl[r] = T.mask + 1; }\n"
      << "        else { sl[r] = slot_of(key, T.shift); k0[r] = T.hot[sl[r] * " << P.agg.hw << "]; } } }\n"
      << "#pragma unroll\n      for (int r = 0; r < R; ++r) { if (!(pass & (1u << r)) || sl[r] == T.mask + 1) continue;\n"
      << "        const uint64_t key = " << V(P.key_reg) << "[r]; uint64_t sx = sl[r], kk = k0[r];\n"
      << "        while (kk != key && kk != kEmptyKey) { sx = (sx + 1) & T.mask; kk = T.hot[sx * " << P.agg.hw << "]; }\n"
      << "        if (kk != key) pass &= ~(1u << r); else sl[r] = sx; }\n";
    emit_loads(s, P.n_early, P.n_in);
    if (P.sink == SINK_PROBE) {
      s << "#pragma unroll\n      for (int r = 0; r < R; ++r) { if (!(pass & (1u << r))) continue;\n"
        << "        unsigned long long* h = reinterpret_cast<unsigned long long*>(T.hot + sl[r] * " << P.agg.hw << ");\n";
      emit_accumulate(s, P, "        ");
      s << "      }\n";
    } else {
      s << "#pragma unroll\n      for (int r = 0; r < R; ++r) { if (!(pass & (1u << r))) continue;\n"
        << "        const uint64_t* cold = T.cold + sl[r] * " << P.agg.cw << ";\n        const uint64_t m = agg_mult(T, sl[r]);\n"
        << "        g0 += m;\n";
      for (int p = 0; p < P.n_sum; ++p) {
        if (P.agg.ps_float[p])
          s << "        g" << 1 + p << " += static_cast<double>(m) * __longlong_as_double(static_cast<long long>("
            << V(P.sum_reg[p]) << "[r]));\n";
        else
          s << "        g" << 1 + p << " += m * " << V(P.sum_reg[p]) << "[r];\n";
      }
      for (int bb = 0; bb < P.agg.nbs; ++bb) {
        if (P.agg.bs_float[bb])
          s << "        g" << 1 + P.n_sum + bb << " += __longlong_as_double(static_cast<long long>(cold[" << 1 + bb << "]));\n";
        else
          s << "        g" << 1 + P.n_sum + bb << " += cold[" << 1 + bb << "];\n";
      }
      s << "      }\n";
    }
    s << "    }\n";
  } else {
    // the semi-join screen runs before the late columns are loaded when its key is an early
    // column (at N > 1 it drops ~90% of the probe side: their late sectors are never read)
    const bool screen_early = P.sink == SINK_MATERIALIZE && (P.semi_kbits != nullptr || P.semi_bloom != nullptr) &&
                              P.semi_key_reg < P.n_early;
    if (screen_early) emit_semi_screen(s, P);
    emit_loads(s, P.n_early, P.n_in);
    if (P.sink == SINK_AGG_SCAN) {  // Q6-analog: rows and sums of the surviving rows
      s << "#pragma unroll\n    for (int r = 0; r < R; ++r) { if (!(pass & (1u << r))) continue;\n      g0 += 1;\n";
      for (int p = 0; p < P.n_sum; ++p) {
        if (P.global_float[1 + p])
          s << "      g" << 1 + p << " += __longlong_as_double(static_cast<long long>(" << V(P.sum_reg[p]) << "[r]));\n";
        else
          s << "      g" << 1 + p << " += " << V(P.sum_reg[p]) << "[r];\n";
      }
      s << "    }\n";
    } else if (P.sink == SINK_KEYBITS) {  // build side straight into the key bitmap
      emit_keybits(s, P);
    } else if (P.sink == SINK_BUILD) {
      s << "    { const AggTableDev& T = P.agg;\n      uint64_t sl[R]; unsigned long long pv[R];\n"
        << "#pragma unroll\n      for (int r = 0; r < R; ++r) { sl[r] = 0; pv[r] = kEmptyKey; if (!(pass & (1u << r))) continue;\n"
        << "        const uint64_t key = " << V(P.key_reg) << "[r];\n"
        << "        if (key == kEmptyKey) { sl[r] = T.mask + 1; continue; }\n"
        << "        sl[r] = slot_of(key, T.shift);\n"
        << "        pv[r] = atomicCAS(reinterpret_cast<unsigned long long*>(T.hot + sl[r] * " << P.agg.hw << "), kEmptyKey, key); }\n"
        << "#pragma unroll\n      for (int r = 0; r < R; ++r) { if (!(pass & (1u << r))) continue;\n"
        << "        const uint64_t key = " << V(P.key_reg) << "[r]; uint64_t sx = sl[r]; bool dup = pv[r] == key;\n"
        << "        if (pv[r] != kEmptyKey && pv[r] != key) sx = agg_insert_from(T, key, (sx + 1) & T.mask, dup);\n"
        << "        agg_count_build(T, key, sx, dup);\n"
        << "        unsigned long long* cold = reinterpret_cast<unsigned long long*>(T.cold + sx * " << P.agg.cw << ");\n";
      for (int bb = 0; bb < P.n_sum; ++bb) {
        if (P.agg.bs_float[bb])
          s << "        atomicAdd(reinterpret_cast<double*>(cold + " << 1 + bb << "), __longlong_as_double(static_cast<long long>("
            << V(P.sum_reg[bb]) << "[r])));\n";
        else
          s << "        atomicAdd(cold + " << 1 + bb << ", static_cast<unsigned long long>(" << V(P.sum_reg[bb]) << "[r]));\n";
      }
      s << "      }\n    }\n";
    } else {  // MATERIALIZE / COUNT
      if (P.sink == SINK_MATERIALIZE && !screen_early) emit_semi_screen(s, P);
      if (P.sink == SINK_MATERIALIZE && P.self_probe && P.nparts > 1) {
        // rows owned by this rank: probe + aggregate in place (two-stage lookup), drop from the shuffle
        s << "    { const AggTableDev& T = P.agg; uint32_t own = 0; uint64_t sl[R], k0[R];\n"
          << "#pragma unroll\n      for (int r = 0; r < R; ++r) if ((pass & (1u << r)) && part_of(" << V(P.part_key_reg)
          << "[r], static_cast<uint32_t>(P.nparts)) == static_cast<uint32_t>(P.self_rank)) own |= 1u << r;\n"
          << "      pass &= ~own;\n"
          << "#pragma unroll\n      for (int r = 0; r < R; ++r) { sl[r] = ~0ULL; k0[r] = 0; if (own & (1u << r)) {\n"
          << "        const uint64_t key = " << V(P.key_reg) << "[r];\n"
          << "        if (key == kEmptyKey) { if (T.cold[(T.mask + 1) * T.cw] == 0) own &= ~(1u << r); else sl[r] = T.mask + 1; }\n"
          << "        else { sl[r] = slot_of(key, T.shift); k0[r] = T.hot[sl[r] * " << P.agg.hw << "]; } } }\n"
          << "#pragma unroll\n      for (int r = 0; r < R; ++r) { if (!(own & (1u << r)) || sl[r] == T.mask + 1) continue;\n"
          << "        const uint64_t key = " << V(P.key_reg) << "[r]; uint64_t sx = sl[r], kk = k0[r];\n"
          << "        while (kk != key && kk != kEmptyKey) { sx = (sx + 1) & T.mask; kk = T.hot[sx * " << P.agg.hw << "]; }\n"
          << "        if (kk != key) own &= ~(1u << r); else sl[r] = sx; }\n"
          << "#pragma unroll\n      for (int r = 0; r < R; ++r) { if (!(own & (1u << r))) continue;\n"
          << "        unsigned long long* h = reinterpret_cast<unsigned long long*>(T.hot + sl[r] * " << P.agg.hw << ");\n";
        emit_accumulate(s, P, "        ");
        s << "      }\n    }\n";
      }
      if (wstage) {
        s << "    { const uint32_t lt = (1u << lane) - 1u;\n"
          << "#pragma unroll\n      for (int r = 0; r < R; ++r) {\n"
          << "        const unsigned b = __ballot_sync(0xffffffffu, (pass >> r) & 1u);\n"
          << "        const int cnt = __popc(b);\n        if (fill + cnt > 128) flush();\n"
          << "        if ((pass >> r) & 1u) { const int pos = fill + __popc(b & lt);\n";
        for (int o = 0; o < P.n_out; ++o)
          s << "          s_stg[warp][" << o << "][pos] = " << out_value(P, o) << ";\n";
        s << "        }\n        fill += cnt;\n      }\n    }\n";
      } else {
      s << "    uint32_t ballots[R];\n#pragma unroll\n    for (int r = 0; r < R; ++r) {\n"
        << "      ballots[r] = __ballot_sync(0xffffffffu, (pass >> r) & 1u);\n"
        << "      if (lane == 0) s_wcnt[warp][r] = __popc(ballots[r]); }\n    __syncthreads();\n"
        << "    if (tid == 0) { uint32_t acc = 0;\n      for (int w = 0; w < " << NW << "; ++w) for (int r = 0; r < R; ++r) { s_woff[w][r] = acc; acc += s_wcnt[w][r]; }\n";
      if (P.sink == SINK_COUNT)
        s << "      P.tile_counts[tile] = acc;\n";
      else if (P.tile_offsets)
        s << "      s_base = P.tile_offsets[tile];\n";
      else
        s << "      s_base = acc ? atomicAdd(P.out_count, static_cast<unsigned long long>(acc)) : 0ULL;\n";
      s << "    }\n    __syncthreads();\n";
      if (P.sink == SINK_MATERIALIZE) {
        s << "    { const uint64_t base = s_base; const uint32_t lt = (1u << lane) - 1u;\n"
          << "#pragma unroll\n      for (int r = 0; r < R; ++r) { if (!((pass >> r) & 1u)) continue;\n"
          << "        const uint64_t pos = base + s_woff[warp][r] + __popc(ballots[r] & lt);\n"
          << "        if (pos >= P.out_cap) continue;\n";
        for (int o = 0; o < P.n_out; ++o) s << "        P.out_col[" << o << "][pos] = " << out_value(P, o) << ";\n";
        s << "      }\n    }\n";
      }
      }
      if (P.sink == SINK_MATERIALIZE) {
        if (part)  // warp-aggregated destination histogram: one shared atomic per (warp, dest)
          s << "#pragma unroll\n    for (int r = 0; r < R; ++r) {\n"
            << "      const bool on = (pass >> r) & 1u;\n"
            << "      const uint32_t d = on ? part_of(" << V(P.part_key_reg) << "[r], static_cast<uint32_t>(P.nparts)) : 0xffffffffu;\n"
            << "      const unsigned peers = __match_any_sync(0xffffffffu, d);\n"
            << "      if (on && lane == __ffs(peers) - 1) atomicAdd(&s_part[d], static_cast<unsigned long long>(__popc(peers)));\n    }\n";
      }
    }
  }
  if (bscan) s << "    __syncthreads();\n";  // s_base / s_woff reuse by the next tile
  s << "    cur_col = pf_col; cur_r0 = pf_r0; cur_rows = pf_rows;\n  }\n";
  if (wstage) s << "  flush();\n";
  if (P.slab) s << "  slab_finish();\n";
  if (P.sink == SINK_KEYBITS)
    s << "  for (int o = 16; o > 0; o >>= 1) kb_rows += __shfl_xor_sync(0xffffffffu, kb_rows, o);\n"
      << "  if (lane == 0 && kb_rows) atomicAdd(P.kb_count, kb_rows);\n";
  if (part)
    s << "  __syncthreads();\n  for (int i = tid; i < P.nparts; i += " << NT << ") if (s_part[i]) atomicAdd(&P.part_counts[i], s_part[i]);\n";
  if (glob) {
    for (int i = 0; i < nglob; ++i) {
      if (P.global_float[i])
        s << "  atomicAdd(reinterpret_cast<double*>(&s_gacc[" << i << "]), g" << i << ");\n";
      else
        s << "  atomicAdd(&s_gacc[" << i << "], g" << i << ");\n";
    }
    s << "  __syncthreads();\n  for (int i = tid; i < " << nglob << "; i += " << NT << ") {\n"
      << "    if (P.global_float[i]) atomicAdd(reinterpret_cast<double*>(&P.global_acc[i]), "
         "__longlong_as_double(static_cast<long long>(s_gacc[i])));\n"
      << "    else atomicAdd(&P.global_acc[i], s_gacc[i]); }\n";
  }
  if (P.slab) s << "  __threadfence_system();  // slab stores visible to the owners before the kernel ends\n";
  s << "}\n";
  return s.str();
}


/// The warp-specialised probe kernel (sm_100a bulk copies + mbarriers). Warp 0 is the producer:
/// one lane streams each 1024-row tile's EARLY columns (predicate + key, the columns every row
/// needs) global -> shared memory with cp.async.bulk into an NS-stage ring, completing on the
/// stage's `full` mbarrier. NG groups of 8 consumer warps take tiles round-robin (group g: tiles
/// g, g + NG, ...), each warp 128 rows of the tile (R = 4 per lane): it copies its rows out of
/// shared memory into registers, releases the stage (`empty` mbarrier, so the producer refills it
/// while this warp works), then evaluates the predicate, probes the rank table (one L2-resident
/// 16-byte record per key), gathers the LATE columns (the sums) from HBM for the surviving rows
/// only and accumulates with atomics. The dense stream is decoupled from the dependent
/// lookup/gather chain, so the HBM stream stays full while consumers wait on L2/HBM latency.
std::string jit_source_staged(const ScanProgram& P) {
  std::ostringstream s;
  const StagedShape sh = staged_shape();
  const int NG = sh.groups, NS = std::max(sh.stages, NG), NE = P.n_early, NIN = P.n_in, nregs = std::max(1, P.n_regs);
  const int CW = sh.warps();  // consumer warps per group (one tile each)
  const int NT = 32 * (1 + CW * NG);
  s << "using namespace psg;\n#define R " << sh.rows << "\n"
    << "extern \"C\" __global__ void __launch_bounds__(" << NT << ", " << sh.ctas
    << ") psg_jit_scan(const __grid_constant__ ScanProgram P, "
       "const Segment* __restrict__ segs, const uint32_t* __restrict__ tile_seg, uint64_t ntiles) {\n"
    << "  extern __shared__ __align__(128) unsigned char smem_raw[];\n"
    << "  uint64_t* stg = reinterpret_cast<uint64_t*>(smem_raw);  // [" << NS << "][" << NE << "][1024]\n"
    << "  __shared__ __align__(8) uint64_t full_bar[" << NS << "], empty_bar[" << NS << "];\n"
    << "  __shared__ const uint64_t* s_col[" << NS << "][" << std::max(1, NIN) << "];\n"
    << "  __shared__ int s_rows[" << NS << "];\n"
    << "  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;\n";
  const bool mat = P.sink == SINK_MATERIALIZE;
  if (mat) {
    // per consumer warp staging rows (dynamic shared memory after the ring)
    s << "  uint64_t* s_stg = stg + " << NS * NE * 1024 << ";\n";
    if (P.nparts > 1)
      s << "  __shared__ unsigned long long s_part[" << kMaxParts << "];\n"
        << "  for (int i = tid; i < " << kMaxParts << "; i += " << NT << ") s_part[i] = 0;\n";
  }
  s << "  if (tid == 0) {\n    for (int i = 0; i < " << NS << "; ++i) { mbar_init(&full_bar[i], 1); mbar_init(&empty_bar[i], " << CW << "); }\n"
    << "    mbar_fence_init();\n  }\n  __syncthreads();\n"
    << "  const uint64_t per_cta = (ntiles + gridDim.x - 1) / gridDim.x;\n"
    << "  const uint64_t t_beg = blockIdx.x * per_cta;\n"
    << "  const uint64_t t_end = t_beg + per_cta < ntiles ? t_beg + per_cta : ntiles;\n"
    << "  if (warp == 0) {  // producer\n"
    << "    if (lane == 0) {\n      const uint64_t pol_stream = l2_evict_first();\n"
    << "      for (uint64_t k = 0; t_beg + k < t_end; ++k) {\n"
    << "        const int st = static_cast<int>(k % " << NS << "); const uint32_t ph = static_cast<uint32_t>((k / " << NS << ") & 1);\n"
    << "        if (k >= " << NS << ") mbar_wait(&empty_bar[st], ph ^ 1u);\n"
    << "        const uint64_t t = t_beg + k;\n        const Segment* sg = segs + __ldg(tile_seg + t);\n"
    << "        const uint64_t r0 = (t - sg->tile_begin) * 1024ULL;\n"
    << "        const int rows = static_cast<int>(min(1024ULL, sg->rows - r0));\n";
  for (int c = NE; c < NIN; ++c) s << "        s_col[st][" << c << "] = sg->col[" << c << "] + r0;\n";
  s << "        s_rows[st] = rows;\n        const uint32_t bytes = (static_cast<uint32_t>(rows) * 8u + 15u) & ~15u;\n"
    << "        mbar_arrive_expect_tx(&full_bar[st], " << NE << "u * bytes);\n";
  for (int c = 0; c < NE; ++c)
    s << "        bulk_g2s(stg + (st * " << NE << " + " << c << ") * 1024, sg->col[" << c << "] + r0, bytes, &full_bar[st], pol_stream);\n";
  s << "      }\n    }\n    return;\n  }\n"
    << "  const uint64_t pol_keep = l2_evict_last(); (void)pol_keep;\n"
    << "  const int cw = (warp - 1) % " << CW << ", grp = (warp - 1) / " << CW << ";\n  const int wrow = cw * (R * 32) + lane;\n";
  if (P.slab && P.sink == SINK_PROBE) emit_slab_prologue(s, P, CW * NG, "warp - 1");
  if (P.sink == SINK_KEYBITS) s << "  unsigned long long kb_rows = 0;\n";
  if (mat) {
    s << "  int fill = 0;\n  auto flush = [&]() {\n    __syncwarp();\n    if (fill == 0) return;\n"
      << "    unsigned long long base = 0;\n    if (lane == 0) base = atomicAdd(P.out_count, static_cast<unsigned long long>(fill));\n"
      << "    base = __shfl_sync(0xffffffffu, base, 0);\n"
      << "    for (int i = lane; i < fill; i += 32) { if (base + i >= P.out_cap) continue;\n";
    for (int o = 0; o < P.n_out; ++o)
      s << "      P.out_col[" << o << "][base + i] = s_stg[((warp - 1) * " << P.n_out << " + " << o << ") * 128 + i];\n";
    s << "    }\n    fill = 0;\n    __syncwarp();\n  };\n";
  }
  s
    << "  for (uint64_t k = grp; t_beg + k < t_end; k += " << NG << ") {\n"
    << "    const int st = static_cast<int>(k % " << NS << "); const uint32_t ph = static_cast<uint32_t>((k / " << NS << ") & 1);\n"
    << "    mbar_wait(&full_bar[st], ph);\n"
    << "    const int nrows = s_rows[st] - cw * (R * 32);\n"
    << "    uint32_t pass = 0;\n#pragma unroll\n    for (int r = 0; r < R; ++r) if (r * 32 + lane < nrows) pass |= 1u << r;\n";
  for (int r = 0; r < nregs; ++r) s << "    uint64_t " << V(r) << "[R] = {};\n";
  for (int c = 0; c < NE; ++c)
    s << "#pragma unroll\n    for (int r = 0; r < R; ++r) if (pass & (1u << r)) " << V(c) << "[r] = stg[(st * " << NE << " + " << c
      << ") * 1024 + wrow + r * 32];\n";
  for (int c = NE; c < NIN; ++c) s << "    const uint64_t* lc" << c << " = s_col[st][" << c << "];\n";
  s << "    __syncwarp();\n    if (lane == 0) mbar_arrive(&empty_bar[st]);  // stage consumed: the producer may refill it\n";
  emit_atoms(s, P);
  emit_joins(s, P);
  auto late = [&] {
    for (int c = NE; c < NIN; ++c)
      s << "#pragma unroll\n      for (int r = 0; r < R; ++r) if (pass & (1u << r)) " << V(c)
        << "[r] = __ldcs(reinterpret_cast<const unsigned long long*>(lc" << c << " + wrow + r * 32));\n";
  };
  if (P.sink == SINK_PROBE) {
    if (P.slab) {
      emit_slab_probe(s, P, late, "warp - 1");
      s << "  }\n  slab_finish();\n  __threadfence_system();  // slab stores visible to the owners before the kernel ends\n}\n";
    } else {
      emit_rank_probe(s, P, late);
      s << "  }\n}\n";
    }
    return s.str();
  }
  if (P.sink == SINK_KEYBITS) {  // late key column for the survivors, then their bits
    late();
    emit_keybits(s, P);
    s << "  }\n"
      << "  for (int o = 16; o > 0; o >>= 1) kb_rows += __shfl_xor_sync(0xffffffffu, kb_rows, o);\n"
      << "  if (lane == 0 && kb_rows) atomicAdd(P.kb_count, kb_rows);\n}\n";
    return s.str();
  }
  // MATERIALIZE: screen -> late columns -> per-warp staging in shared memory, flushed 128 rows at
  // a time with one global atomic; destination histogram in shared memory (part)
  const bool part = P.nparts > 1;
  const bool screen_early = (P.semi_kbits != nullptr || P.semi_bloom != nullptr) && P.semi_key_reg < NE;
  if (screen_early) emit_semi_screen(s, P);
  late();
  if (!screen_early) emit_semi_screen(s, P);
  s << "    { const uint32_t lt = (1u << lane) - 1u;\n"
    << "#pragma unroll\n      for (int r = 0; r < R; ++r) {\n"
    << "        const unsigned b = __ballot_sync(0xffffffffu, (pass >> r) & 1u);\n"
    << "        const int cnt = __popc(b);\n        if (fill + cnt > 128) flush();\n"
    << "        if ((pass >> r) & 1u) { const int pos = fill + __popc(b & lt);\n";
  for (int o = 0; o < P.n_out; ++o)
    s << "          s_stg[((warp - 1) * " << P.n_out << " + " << o << ") * 128 + pos] = " << out_value(P, o) << ";\n";
  s << "        }\n        fill += cnt;\n      }\n    }\n";
  if (part)
    s << "#pragma unroll\n    for (int r = 0; r < R; ++r) {\n"
      << "      const bool on = (pass >> r) & 1u;\n"
      << "      const uint32_t d = on ? part_of(" << V(P.part_key_reg) << "[r], static_cast<uint32_t>(P.nparts)) : 0xffffffffu;\n"
      << "      const unsigned peers = __match_any_sync(0xffffffffu, d);\n"
      << "      if (on && lane == __ffs(peers) - 1) atomicAdd(&s_part[d], static_cast<unsigned long long>(__popc(peers)));\n    }\n";
  s << "  }\n  flush();\n";
  if (part)
    s << "  asm volatile(\"bar.sync 1, " << 32 * CW * NG << ";\" ::: \"memory\");  // consumers only (the producer exited)\n"
      << "  for (int i = tid - 32; i < P.nparts; i += " << 32 * CW * NG << ") if (s_part[i]) atomicAdd(&P.part_counts[i], s_part[i]);\n";
  s << "}\n";
  return s.str();
}

namespace {

/// NVRTC: CUDA C++ -> sm_100a cubin. Returns false (with the log) on failure.
bool nvrtc_cubin(const std::string& body, std::string& cubin, std::string& log) {
  const std::string src = std::string(kDeviceCommonSrc) + "\n" + body;
  nvrtcProgram prog;
  if (nvrtcCreateProgram(&prog, src.c_str(), "psg_jit_scan.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS) {
    log = "nvrtcCreateProgram failed";
    return false;
  }
  const char* opts[] = {"--gpu-architecture=sm_100a", "-std=c++17", "-lineinfo", "--restrict"};
  const nvrtcResult r = nvrtcCompileProgram(prog, 4, opts);
  size_t n = 0;
  nvrtcGetProgramLogSize(prog, &n);
  log.assign(n, '\0');
  if (n) nvrtcGetProgramLog(prog, log.data());
  if (r != NVRTC_SUCCESS) {
    nvrtcDestroyProgram(&prog);
    return false;
  }
  nvrtcGetCUBINSize(prog, &n);
  cubin.assign(n, '\0');
  nvrtcGetCUBIN(prog, cubin.data());
  nvrtcDestroyProgram(&prog);
  return true;
}

Compiled compile(const std::string& body, int device, int block, int smem) {
  Compiled c;
  c.block = block;
  c.smem = smem;
  const auto t0 = std::chrono::steady_clock::now();
  std::string cubin, log;
  if (const char* dir = std::getenv("PSG_JIT_DUMP")) {
    // diagnostics: the generated kernel source, for offline SASS inspection (nvcc -cubin)
    static int seq = 0;
    const std::string path = std::string(dir) + "/psg_jit_" + std::to_string(getpid()) + "_" + std::to_string(seq++) + ".cu";
    if (FILE* f = std::fopen(path.c_str(), "w")) {
      std::fwrite(body.data(), 1, body.size(), f);
      std::fclose(f);
    }
  }
  if (!nvrtc_cubin(body, cubin, log)) {
    std::fprintf(stderr, "[psg] NVRTC compile failed (falling back to the interpreter kernel):\n%s\n", log.c_str());
    return c;
  }
  if (cudaLibraryLoadData(&c.lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0) != cudaSuccess) {
    cudaGetLastError();
    return c;
  }
  if (cudaLibraryGetKernel(&c.kern, c.lib, "psg_jit_scan") != cudaSuccess) {
    cudaGetLastError();
    return c;
  }
  if (c.smem > 0 &&  // (static + dynamic > 48 KB needs the opt-in even when dynamic alone does not)
      cudaFuncSetAttribute(reinterpret_cast<const void*>(c.kern), cudaFuncAttributeMaxDynamicSharedMemorySize, c.smem) !=
          cudaSuccess) {
    cudaGetLastError();
    return c;
  }
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, reinterpret_cast<const void*>(c.kern), c.block, c.smem) !=
          cudaSuccess ||
      per_sm < 1) {
    cudaGetLastError();
    per_sm = 4;
  }
  c.per_sm = per_sm;
  c.ok = true;
  if (std::getenv("PSG_TRACE")) {
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, reinterpret_cast<const void*>(c.kern));
    std::fprintf(stderr, "[psg] jit kernel: %d regs, %zu B local, %d CTAs/SM, %d threads, %d B dynamic smem (%zu B source)\n",
                 fa.numRegs, static_cast<size_t>(fa.localSizeBytes), per_sm, c.block, c.smem, body.size());
  }
  g_compile_s += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  ++g_compiles;
  (void)device;
  return c;
}

}  // namespace

void fused_scan(const ScanProgram& P, const Segment* d_segs, const uint32_t* d_tile_seg, int nsegs, uint64_t ntiles,
                cudaStream_t stream) {
  if (ntiles == 0 || nsegs == 0) return;
  if (jit_enabled()) {
    int dev = 0;
    cudaGetDevice(&dev);
    const std::string body = jit_source(P);
    Compiled c;
    {
      std::lock_guard<std::mutex> lk(g_mu);
      auto key = std::make_pair(dev, body);
      auto it = g_cache.find(key);
      if (it == g_cache.end()) {
        int block = jit_block(P), smem = 0;
        if (staged_probe(P)) {
          const StagedShape sh = staged_shape();
          block = 32 * (1 + sh.warps() * sh.groups);
          smem = std::max(sh.stages, sh.groups) * P.n_early * 1024 * 8;
          if (P.sink == SINK_MATERIALIZE) smem += sh.warps() * sh.groups * P.n_out * 128 * 8;
        }
        it = g_cache.emplace(key, compile(body, dev, block, smem)).first;
      }
      c = it->second;
    }
    if (c.ok) {
      int sms = 148;
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      uint64_t grid = static_cast<uint64_t>(sms) * c.per_sm;
      if (grid > ntiles) grid = ntiles;
      void* args[] = {const_cast<ScanProgram*>(&P), const_cast<Segment**>(&d_segs), const_cast<uint32_t**>(&d_tile_seg),
                      &ntiles};
      count_external_launch();
      PSG_CUDA(cudaLaunchKernel(reinterpret_cast<const void*>(c.kern), dim3(static_cast<unsigned>(grid)), dim3(c.block),
                                args, static_cast<size_t>(c.smem), stream));
      return;
    }
  }
  if (P.remote) throw Error(PSG_ERR_INTERNAL, "the fused NVLink path needs the query compiler (PSG_JIT)");
  if (P.self_probe || P.pack_n || P.unpack_n || P.agg.npacked || P.agg.krank || P.slab || P.sink == SINK_KEYBITS)
    throw Error(PSG_ERR_INTERNAL,
                "owner probe / packed rows / packed accumulators / rank-indexed table need the query compiler (PSG_JIT)");
  launch_scan(P, d_segs, d_tile_seg, nsegs, ntiles, stream);
}

bool jit_available() { return jit_enabled(); }

int jit_selftest(std::string& log) {
  // Representative program structures: every sink, int/float atoms, a local join with payload,
  // Bloom-screened probe, partition histogram, ordered compaction, global aggregate.
  std::vector<ScanProgram> progs;
  auto base = [] {
    ScanProgram p;
    std::memset(&p, 0, sizeof p);
    p.n_in = 4;
    p.n_pred = 1;
    p.n_early = 2;
    p.n_regs = 4;
    p.n_atoms = 2;
    p.atoms[0] = AtomDesc{0, 5, 0, 0, 19950315};
    p.atoms[1] = AtomDesc{0, 3, 0, 0, 7};
    p.key_reg = 1;
    p.part_key_reg = -1;
    return p;
  };
  for (int sink : {SINK_MATERIALIZE, SINK_BUILD, SINK_PROBE, SINK_PROBE_GLOBAL, SINK_COUNT, SINK_AGG_SCAN}) {
    ScanProgram p = base();
    p.sink = sink;
    p.n_sum = 2;
    p.sum_reg[0] = 2;
    p.sum_reg[1] = 3;
    p.agg.hw = 4;
    p.agg.cw = 2;
    p.agg.nbs = 1;
    p.agg.ps_float[1] = 1;
    p.agg.bs_float[0] = 1;
    p.global_float[2] = 1;
    p.global_float[3] = 1;
    p.n_out = 3;
    p.out_reg[0] = 1, p.out_reg[1] = 2, p.out_reg[2] = 3;
    if (sink == SINK_PROBE) p.agg.bloom = reinterpret_cast<uint32_t*>(16);
    if (sink == SINK_MATERIALIZE) {
      p.nparts = 4;
      p.part_key_reg = 1;
      p.semi_bloom = reinterpret_cast<const uint32_t*>(16);
      p.semi_key_reg = 1;
    }
    progs.push_back(p);
    if (sink == SINK_MATERIALIZE) {  // + in-place probe of the rows this rank owns
      p.self_probe = 1;
      p.self_rank = 2;
      p.key_reg = 1;
      progs.push_back(p);
      p.pack_n = 3;  // + bit-packed output rows
      p.pack_reg[0] = 1, p.pack_reg[1] = 2, p.pack_reg[2] = 3;
      p.n_out = 1;
      progs.push_back(p);
    }
    if (sink == SINK_MATERIALIZE) {  // exact global semi-join bitmap instead of the Blooms
      ScanProgram q = p;
      q.semi_bloom = nullptr;
      q.semi_kbits = reinterpret_cast<const uint32_t*>(16);
      progs.push_back(q);
      q.self_probe = 0;  // the warp-specialised bulk-copy partitioning scan (packed rows)
      q.staged_ok = 1;
      progs.push_back(q);
      q.pack_n = 0;  // ... and with plain multi-column rows, no partition
      q.n_out = 3;
      q.nparts = 0;
      q.semi_kbits = nullptr;
      progs.push_back(q);
    }
    if (sink == SINK_PROBE) {  // packed accumulators: hits + sum 0 in word 1, sum 1 (float) alone
      ScanProgram q = p;
      q.agg.npacked = 1;
      q.agg.packed_shift[0] = 30;
      q.agg.packed_shift[1] = -1;
      progs.push_back(q);
    }
    if (sink == SINK_PROBE) {  // exact membership bitmap instead of the Bloom filter
      ScanProgram q = p;
      q.agg.kbits = reinterpret_cast<uint32_t*>(16);
      progs.push_back(q);
      q.agg.krank = reinterpret_cast<const uint32_t*>(16);  // rank-indexed table
      progs.push_back(q);
      q.agg.krec = reinterpret_cast<const unsigned long long*>(16);  // + interleaved rank records
      progs.push_back(q);
      q.staged_ok = 1;  // the warp-specialised bulk-copy probe
      q.agg.npacked = 1;
      q.agg.packed_shift[0] = 30;
      q.agg.packed_shift[1] = -1;
      progs.push_back(q);
      q.bkt = reinterpret_cast<uint64_t*>(16);  // + bucketed aggregation
      q.agg.ps_float[1] = 0;
      progs.push_back(q);
      q.slab = 1;  // + peer-slab shuffle: global screen, packed rows to the owners' slabs
      q.nparts = 4;
      q.self_rank = 1;
      q.semi_kbits = reinterpret_cast<const uint32_t*>(16);
      q.semi_key_reg = 1;
      q.pack_n = 3;
      q.pack_reg[0] = 1, q.pack_reg[1] = 2, q.pack_reg[2] = 3;
      q.slab_grec = reinterpret_cast<const unsigned long long*>(16);
      progs.push_back(q);
      q.staged_ok = 0;  // ... in the register kernel
      progs.push_back(q);
      q.staged_ok = 1;  // two ranks: the ballot-based put
      q.nparts = 2;
      q.self_rank = 1;
      progs.push_back(q);
    }
    if (sink == SINK_PROBE) {  // consuming packed rows
      ScanProgram q = p;
      q.unpack_n = 3;
      q.n_in = 1, q.n_pred = 0, q.n_early = 1, q.n_regs = 4, q.n_atoms = 0;
      q.key_reg = 1;
      progs.push_back(q);
    }
  }
  {
    ScanProgram p = base();  // build side straight into the key bitmap
    p.sink = SINK_KEYBITS;
    progs.push_back(p);
    p.kb_flag = reinterpret_cast<unsigned int*>(16);  // ... with the in-kernel duplicate flag
    progs.push_back(p);
    p.kb_flag = nullptr;
    p.staged_ok = 1;  // ... warp-specialised
    progs.push_back(p);
  }
  {
    ScanProgram p = base();  // orders-like: filter, local join with payload, materialise
    p.sink = SINK_MATERIALIZE;
    p.n_in = 3;
    p.n_regs = 5;
    p.n_joins = 1;
    p.joins[0].key_reg = 1;
    p.joins[0].t.npayload = 2;
    p.joins[0].payload_reg[0] = 3;
    p.joins[0].payload_reg[1] = 4;
    p.atoms[1] = AtomDesc{0, 1, 1, 0, 0};
    p.n_out = 2;
    p.out_reg[0] = 2, p.out_reg[1] = 4;
    p.tile_offsets = reinterpret_cast<const uint64_t*>(16);
    progs.push_back(p);
    p.joins[0].t.npayload = 0;  // semi-join through a membership bitmap
    p.joins[0].t.bitmap = reinterpret_cast<const uint32_t*>(16);
    p.out_reg[1] = 2;
    progs.push_back(p);
  }
  for (int sink : {SINK_BUILD, SINK_PROBE}) {
    ScanProgram p = base();
    p.sink = sink;
    p.remote = 1;
    p.nparts = 4;
    p.n_sum = 2;
    p.sum_reg[0] = 2;
    p.sum_reg[1] = 3;
    p.agg.hw = 4;
    p.agg.cw = 2;
    p.agg.ps_float[1] = 1;
    p.agg.bs_float[1] = 1;
    p.semi_bloom = reinterpret_cast<const uint32_t*>(16);
    p.semi_key_reg = 1;
    progs.push_back(p);
  }
  int failures = 0;
  int seq = 0;
  for (auto& p : progs) {
    std::string cubin, l;
    const std::string src = jit_source(p);
    if (!nvrtc_cubin(src, cubin, l) || cubin.empty()) {
      ++failures;
      log += "sink " + std::to_string(p.sink) + ": " + l + "\n";
    } else if (const char* dir = std::getenv("PSG_JIT_DUMP")) {  // cubins + sources for cuobjdump -sass
      const std::string base = std::string(dir) + "/selftest_" + std::to_string(seq) + (staged_probe(p) ? "_staged" : "");
      if (FILE* f = std::fopen((base + ".cubin").c_str(), "wb")) {
        std::fwrite(cubin.data(), 1, cubin.size(), f);
        std::fclose(f);
      }
      if (FILE* f = std::fopen((base + ".cu").c_str(), "w")) {
        std::fwrite(src.data(), 1, src.size(), f);
        std::fclose(f);
      }
    }
    ++seq;
  }
  return failures;
}

JitStats jit_stats() {
  std::lock_guard<std::mutex> lk(g_mu);
  return JitStats{g_compiles, g_compile_s, jit_enabled()};
}

}  // namespace psg
