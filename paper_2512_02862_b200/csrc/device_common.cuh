// Device data structures + hash-table primitives shared by the nvcc-compiled kernels (kernels.cu)
// and the NVRTC-compiled per-plan kernels (jit.cpp embeds this file verbatim), so both agree on
// layout and hashing bit for bit.
#pragma once

#ifdef __CUDACC_RTC__
typedef unsigned long long uint64_t;
typedef long long int64_t;
typedef unsigned int uint32_t;
typedef int int32_t;
#else
#include <cstdint>
#endif

namespace psg {

constexpr uint64_t kEmptyKey = 0x8000000000000000ULL;  // INT64_MIN; real INT64_MIN keys use the spill slot
constexpr int kMaxIn = 16;
constexpr int kMaxAtoms = 8;
constexpr int kMaxJoins = 4;
constexpr int kMaxPayload = 8;
constexpr int kMaxRegs = 26;  // interpreter smem = n_regs * 4 rows * 256 threads * 8 B <= 208 KiB
constexpr int kMaxOut = 16;
constexpr int kMaxSums = 8;
constexpr int kMaxParts = 64;
constexpr int kMaxSlabPeers = 16;  // peer-slab shuffle: GPUs of one box
constexpr int kBlock = 256;
constexpr int kBucketSlots = 2048;  // rank-table slots per aggregation bucket (shared-memory slice)
constexpr int kBucketBits = 11;
constexpr int kRowsPerThread = 4;
constexpr uint64_t kSlotMul = 0xD6E8FEB86659FD93ULL;   // table slot = (k * kSlotMul) >> shift
constexpr uint64_t kBloomMul = 0xA24BAED4963EE407ULL;  // bloom word/bits from (k * kBloomMul)
constexpr uint64_t kPartMul = 0x9E3779B97F4A7C15ULL;   // partition_of, hashing.hpp:26-28

// SINK_AGG_SCAN: global aggregate straight off the scan (no probe) - the Q6-analog local plans.
enum SinkKind : int {
  SINK_MATERIALIZE = 0,
  SINK_BUILD = 1,
  SINK_PROBE = 2,
  SINK_PROBE_GLOBAL = 3,
  SINK_COUNT = 4,
  SINK_AGG_SCAN = 5,
  SINK_KEYBITS = 6
};

/// One row group (or one received/materialised run): rows + a device pointer per input column.
struct Segment {
  const uint64_t* col[kMaxIn];
  uint64_t rows;
  uint64_t tile_begin;  // first tile index of this segment (prefix over segments)
};

struct AtomDesc {
  int32_t reg;
  int32_t op;        // CmpOp: 0 <, 1 <=, 2 ==, 3 !=, 4 >=, 5 >
  int32_t is_float;  // compare as double (column type Float64)
  int32_t pad;
  uint64_t lit;      // int64 literal or double bits (already cast per literal_as<T>)
};

/// CSR hash table of a replicated build side (local join). Slots [0,cap) linear-probed by key;
/// slot cap is the spill slot for key == kEmptyKey.
struct LocalTableDev {
  uint64_t* keys;
  uint32_t* cnt;
  uint32_t* start;
  uint64_t mask;
  const uint64_t* payload[kMaxPayload];  // CSR-ordered payload columns (needed ones only)
  int32_t npayload;
  int32_t shift;  // 64 - log2(cap)
  // Dense unique keys with no payload needed (a semi-join, e.g. customer(seg) in Q3): membership
  // bitmap over [bmin, bmin + brange) instead of the hash table (bitmap != nullptr).
  const uint32_t* bitmap;
  int64_t bmin;
  uint64_t brange;
};

struct JoinDesc {
  LocalTableDev t;
  int32_t key_reg;
  int32_t payload_reg[kMaxPayload];  // destination register of each payload column
};

/// Shuffle-join aggregation table (group key == join key, pipeline.cpp:191-195):
///   hot[slot*hw + 0] = key, +1 = probe hits, +2.. = probe-side sums
///   cold[slot*cw + 0] = build multiplicity m, +1.. = build-side sums
/// slot == cap is the spill slot of key == kEmptyKey (occupied iff m > 0).
struct AggTableDev {
  uint64_t* hot;
  uint64_t* cold;
  uint32_t* bloom;   // optional blocked Bloom filter over the keys (nullptr = none)
  uint64_t mask;
  uint64_t bloom_mask;  // number of 32-bit words - 1
  int32_t hw, cw;
  int32_t nps, nbs;  // probe-side / build-side sums
  int32_t ps_float[kMaxSums];
  int32_t bs_float[kMaxSums];
  int32_t shift;        // 64 - log2(cap)
  int32_t bloom_shift;  // 64 - log2(bloom words)
  unsigned int* dups;   // set to 1 when a build key repeats (nullptr: unknown, assume repeats)
  // Dense build keys: exact membership bitmap over [kmin, kmin + krange) instead of the Bloom
  // filter (kbits != nullptr; set by the build, tested by the probe).
  uint32_t* kbits;
  int64_t kmin;
  uint64_t krange;
  // Bit-packed accumulators (int probe-side sums bounded by the footer zone maps): word 1 of a hot
  // slot holds the hit count in its low bits (hits_mask) and every packed sum p, accumulated as
  // value - packed_min[p], in the field at packed_shift[p] (packed_shift < 0: own word 2 + p).
  // One atomicAdd per hit covers them all; word 1 != 0 still means "hit".
  int32_t npacked;
  int32_t packed_shift[kMaxSums];
  uint64_t packed_mask[kMaxSums];
  int64_t packed_min[kMaxSums];
  uint64_t hits_mask;
  // Rank-indexed table (one GPU, unique dense build keys; krank != nullptr): the slot of a key is
  // its rank among the build keys, krank[w] + popc(kbits64[w] below the key's bit) for 64-bit
  // bitmap word w, so slots [0, mask] are all occupied in key order and nothing is hashed.
  const uint32_t* krank;
  // {kbits64[w], krank[w]} interleaved per 64-key word (16 B): membership and rank of a key in ONE
  // L2 sector (nullptr: use kbits/krank)
  const unsigned long long* krec;
};

/// Hit count and probe-side sum p of a hot slot (decodes the packed accumulator).
__device__ __forceinline__ uint64_t agg_hits(const AggTableDev& t, const uint64_t* h) {
  return t.npacked ? (h[1] & t.hits_mask) : h[1];
}
__device__ __forceinline__ uint64_t agg_psum(const AggTableDev& t, const uint64_t* h, int p, uint64_t hits) {
  if (t.npacked && t.packed_shift[p] >= 0)
    return ((h[1] >> t.packed_shift[p]) & t.packed_mask[p]) + hits * static_cast<uint64_t>(t.packed_min[p]);
  return h[2 + p];
}

/// One rank's aggregation-table arrays as mapped into this process (CUDA IPC symmetric heap).
struct AggPeer {
  uint64_t* hot;
  uint64_t* cold;
  uint32_t* bloom;
  uint64_t pad;
};

struct ScanProgram {
  int32_t n_in;        // regs [0,n_in) load from Segment::col
  int32_t n_pred;      // regs [0,n_pred) are loaded for every row (predicate columns)
  int32_t n_early;     // regs [n_pred,n_early) load after the predicate, before joins/probe
  int32_t n_regs;      // total registers (inputs + join payloads)
  int32_t n_atoms;
  int32_t n_joins;
  AtomDesc atoms[kMaxAtoms];
  JoinDesc joins[kMaxJoins];
  int32_t sink;
  // SINK_MATERIALIZE / SINK_COUNT
  int32_t n_out;
  int32_t out_reg[kMaxOut];
  uint64_t* out_col[kMaxOut];
  uint64_t out_cap;
  unsigned long long* out_count;        // atomic reservation counter (unordered tiles)
  const uint64_t* tile_offsets;         // ordered mode: exclusive prefix of tile counts
  unsigned long long* tile_counts;      // SINK_COUNT output
  int32_t nparts;                       // >1: histogram of partition_of(reg[part_key_reg])
  int32_t part_key_reg;
  unsigned long long* part_counts;
  // SINK_BUILD / SINK_PROBE / SINK_PROBE_GLOBAL
  int32_t key_reg;
  int32_t n_sum;
  int32_t sum_reg[kMaxSums];            // probe: probe-side sums; build: build-side sums
  AggTableDev agg;
  unsigned long long* global_acc;       // SINK_PROBE_GLOBAL: [rows, probe sums..., build sums...]; AGG_SCAN: [rows, sums...]
  int32_t global_float[2 * kMaxSums + 1];
  // Semi-join pre-filter of a partitioned probe side (MATERIALIZE with nparts > 1): nparts
  // concatenated Bloom filters, filter d over the build keys owned by rank d. A row whose key is
  // certainly absent on its owner is dropped before it is shuffled.
  const uint32_t* semi_bloom;
  uint64_t semi_words;
  int32_t semi_shift;
  int32_t semi_key_reg;
  // MATERIALIZE with nparts > 1: rows this rank owns (part_of(key) == self_rank) are probed and
  // aggregated into `agg` in place (grouped aggregate, key_reg / n_sum / sum_reg) and never
  // materialised or shuffled - only rows owned by other ranks leave the kernel.
  int32_t self_probe;
  int32_t self_rank;
  // Exact semi-join: one global membership bitmap of every rank's build keys over
  // [semi_kmin, semi_kmin + semi_krange) (replaces semi_bloom when set).
  const uint32_t* semi_kbits;
  int64_t semi_kmin;
  uint64_t semi_krange;
  // Bit-packed shuffle rows: MATERIALIZE with pack_n > 0 writes ONE word per row (out column 0),
  // sum_k (reg[pack_reg[k]] - pack_min[k]) << pack_shift[k]; a program with unpack_n > 0 first
  // expands register 0 into registers 1..unpack_n (value = pack_min + (w >> shift & mask)).
  int32_t pack_n, unpack_n;
  int32_t pack_reg[kMaxOut];
  int32_t pack_shift[kMaxOut];
  int64_t pack_min[kMaxOut];
  uint64_t pack_mask[kMaxOut];
  // Fused NVLink path (SINK_BUILD / SINK_PROBE with remote = 1): every row's table operation goes
  // to the owner rank part_of(key) directly in its (peer-mapped) table; tables are symmetric so
  // mask/shift/hw/cw come from `agg`, only the base pointers differ per rank.
  const AggPeer* peers;
  int32_t remote;
  // Bucketed aggregation (rank-indexed table, SINK_PROBE): a surviving row is appended as ONE word
  // to the bucket of its slot (slot >> kBucketBits): slot & (kBucketSlots - 1) in the low bits,
  // then every probe sum k as (v - bkt_min[k]) & bkt_mask[k] at bkt_shift[k]. k_bucket_agg then
  // folds each bucket in shared memory and adds it to the hot slots once, so the table's random
  // read-modify-writes never go to HBM. A full bucket spills to the overflow list below.
  // Each bucket is split into 2^bkt_sub_bits sub-lists (a row goes to sub-list threadIdx & (S-1)):
  // S x more append counters - the L2 serves atomics on few distinct words far slower (measured:
  // 42 G/s on 3.6 K counters vs 142 G/s on 64 K, profiles/r2_atomic_probe.txt).
  uint64_t* bkt;             // [nbuckets << bkt_sub_bits][bkt_cap]
  unsigned int* bkt_fill;    // [nbuckets << bkt_sub_bits] appended entries (may exceed bkt_cap: overflowed)
  uint32_t bkt_cap;
  int32_t bkt_sub_bits;
  int32_t bkt_shift[kMaxSums];
  uint64_t bkt_mask[kMaxSums];
  int64_t bkt_min[kMaxSums];
  // a full bucket's rows go to one overflow list: {full slot, entry word} pairs; beyond its
  // capacity the engine re-runs the query without buckets (bkt_ovf_count > bkt_ovf_cap)
  uint64_t* bkt_ovf;
  unsigned int* bkt_ovf_count;
  uint32_t bkt_ovf_cap;
  // SINK_KEYBITS: a build side that only feeds the rank-indexed table sets bit (key - kb_min) of
  // kb_bits for every surviving row instead of materialising it; kb_flag |= 1 when the bit was
  // already set (a duplicate key), |= 2 for a key outside [kb_min, kb_min + kb_range); kb_count
  // counts the rows.
  uint32_t* kb_bits;
  int64_t kb_min;
  uint64_t kb_range;
  unsigned int* kb_flag;
  unsigned long long* kb_count;
  // Peer-slab shuffle (SINK_PROBE at N > 1, slab = 1): after the global semi-join screen, a row
  // owned by rank d != self_rank is bit-packed (pack_*) and stored straight into this rank's
  // region of d's receive slab through NVLink (slab_dst[d], peer-mapped), at a position reserved
  // with one atomic per (warp, destination) on slab_cnt[d]; rows this rank owns are probed in
  // place. No materialisation, no count exchange, no NCCL on the data path.
  uint64_t* slab_dst[kMaxSlabPeers];
  unsigned long long* slab_cnt;
  uint64_t slab_cap;
  int32_t slab;
  // {global key-bitmap word, rank of this rank's first own key in the word} per 64 keys: ONE
  // 16-byte lookup screens every row and gives an own row its slot (own keys below it in the word
  // are the global bits whose key this rank owns - counted by hashing only those few keys)
  const unsigned long long* slab_grec;
  // the engine guarantees 16-byte aligned column chunks and readable padding past each chunk's
  // end (PSTO batches, staged images): the query compiler may then stream the early columns into
  // shared memory with bulk copies (the warp-specialised probe, jit.cpp)
  int32_t staged_ok;
};
static_assert(sizeof(ScanProgram) <= 4096, "ScanProgram is a kernel parameter (4 KB limit)");

#if defined(__CUDACC__) || defined(__CUDACC_RTC__)
/// partition_of (hashing.hpp:26-37): ((k * 0x9E3779B97F4A7C15) >> 13) % n
__device__ __forceinline__ uint32_t part_of(uint64_t k, uint32_t n) {
  const uint64_t h = (k * kPartMul) >> 13;
  // power-of-two node counts (the usual 2/4/8 GPUs) avoid the 64-bit remainder (~100 instructions)
  return (n & (n - 1)) == 0 ? static_cast<uint32_t>(h & (n - 1)) : static_cast<uint32_t>(h % n);
}
__device__ __forceinline__ uint64_t slot_of(uint64_t key, int shift) { return (key * kSlotMul) >> shift; }

__device__ __forceinline__ bool cmp_i(int64_t a, int op, int64_t b) {
  switch (op) {
    case 0: return a < b;
    case 1: return a <= b;
    case 2: return a == b;
    case 3: return a != b;
    case 4: return a >= b;
    default: return a > b;
  }
}
__device__ __forceinline__ bool cmp_f(double a, int op, double b) {
  switch (op) {  // IEEE semantics (NaN compares false except !=)
    case 0: return a < b;
    case 1: return a <= b;
    case 2: return a == b;
    case 3: return a != b;
    case 4: return a >= b;
    default: return a > b;
  }
}

__device__ __forceinline__ uint32_t bloom_bits(uint64_t h2, int bshift) {
  return (1u << ((h2 >> (bshift - 5)) & 31)) | (1u << ((h2 >> (bshift - 10)) & 31)) |
         (1u << ((h2 >> (bshift - 15)) & 31));
}
/// Rank-indexed table: the slot of key (a build key) from the 64-bit view of the key bitmap.
__device__ __forceinline__ uint64_t agg_rank_slot(const AggTableDev& t, uint64_t key) {
  const uint64_t d = key - static_cast<uint64_t>(t.kmin);
  const uint64_t w = __ldg(reinterpret_cast<const unsigned long long*>(t.kbits) + (d >> 6));
  return __ldg(t.krank + (d >> 6)) + __popcll(w & ((1ULL << (d & 63)) - 1ULL));
}

__device__ __forceinline__ bool agg_kbit(const AggTableDev& t, uint64_t key) {
  const uint64_t d = key - static_cast<uint64_t>(t.kmin);
  return d < t.krange && ((__ldg(t.kbits + (d >> 5)) >> (d & 31)) & 1u);
}
__device__ __forceinline__ bool bloom_maybe(const AggTableDev& t, uint64_t key) {
  if (t.kbits != nullptr) return agg_kbit(t, key);
  if (t.bloom == nullptr) return true;
  const uint64_t h2 = key * kBloomMul;
  const uint32_t m = bloom_bits(h2, t.bloom_shift);
  const uint32_t w = __ldg(t.bloom + (h2 >> t.bloom_shift));
  return (w & m) == m;
}

/// Claims key's slot from s on; `dup` = the key was already present (another build row).
// ---- TMA bulk copies (cp.async.bulk, sm_90+) completing on a shared-memory mbarrier ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
/// L2 policies: streamed column data is evict-first so it never displaces the L2-resident Bloom
/// filters and hash-table lines that the probes hit.
__device__ __forceinline__ uint64_t l2_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint32_t ldg_keep_u32(const uint32_t* p, uint64_t policy) {
  uint32_t v;
  asm volatile("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(policy));
  return v;
}
__device__ __forceinline__ uint64_t ldg_keep_u64(const void* p, uint64_t policy) {
  uint64_t v;
  asm volatile("ld.global.nc.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(v) : "l"(p), "l"(policy));
  return v;
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
/// Makes mbarrier.init visible to the async (bulk-copy) proxy before the first copy.
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n\tfence.proxy.async.shared::cta;" ::: "memory");
}
/// 16-byte L2-resident record (evict_last policy), e.g. the rank table's {bits, rank} word.
__device__ __forceinline__ void ldg_keep_v2u64(const unsigned long long* p, uint64_t policy, uint64_t& a, uint64_t& b) {
  asm volatile("ld.global.nc.L2::cache_hint.v2.u64 {%0, %1}, [%2], %3;" : "=l"(a), "=l"(b) : "l"(p), "l"(policy));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  const uint32_t a = smem_u32(bar);
  while (!done)
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
}

/// Semi-join test: false only when key is certainly not a build key of its owner rank.
__device__ __forceinline__ bool semi_maybe(const ScanProgram& P, uint64_t key) {
  if (key == kEmptyKey) return true;  // the spill key is never in the filters
  if (P.semi_kbits != nullptr) {
    const uint64_t d = key - static_cast<uint64_t>(P.semi_kmin);
    return d < P.semi_krange && ((__ldg(P.semi_kbits + (d >> 5)) >> (d & 31)) & 1u);
  }
  const uint64_t h2 = key * kBloomMul;
  const uint32_t d = part_of(key, static_cast<uint32_t>(P.nparts));
  const uint32_t w = __ldg(P.semi_bloom + d * P.semi_words + (h2 >> P.semi_shift));
  const uint32_t m = bloom_bits(h2, P.semi_shift);
  return (w & m) == m;
}

__device__ __forceinline__ uint64_t agg_insert_from(const AggTableDev& t, uint64_t key, uint64_t s, bool& dup) {
  while (true) {
    unsigned long long* kp = reinterpret_cast<unsigned long long*>(t.hot + s * t.hw);
    const unsigned long long prev = atomicCAS(kp, kEmptyKey, key);
    if (prev == kEmptyKey || prev == key) {
      dup = prev == key;
      return s;
    }
    s = (s + 1) & t.mask;
  }
}
/// Build multiplicity m of an occupied slot: cold[0] counts duplicates (m - 1) so unique build
/// keys never touch the cold array; the kEmptyKey spill slot counts m directly.
__device__ __forceinline__ uint64_t agg_mult(const AggTableDev& t, uint64_t slot) {
  const uint64_t c = t.cold[slot * t.cw];
  return slot == t.mask + 1 ? c : c + 1;
}
/// Records one build row of key in slot (after agg_insert_from): duplicate count + Bloom bits.
__device__ __forceinline__ void agg_count_build(const AggTableDev& t, uint64_t key, uint64_t slot, bool dup) {
  if (slot == t.mask + 1 || dup) {
    atomicAdd(reinterpret_cast<unsigned long long*>(t.cold + slot * t.cw), 1ULL);
    if (dup && t.dups != nullptr) *t.dups = 1u;
  } else if (t.kbits != nullptr) {
    const uint64_t d = key - static_cast<uint64_t>(t.kmin);
    atomicOr(t.kbits + (d >> 5), 1u << (d & 31));
  } else if (t.bloom != nullptr) {
    const uint64_t h2 = key * kBloomMul;
    atomicOr(t.bloom + (h2 >> t.bloom_shift), bloom_bits(h2, t.bloom_shift));
  }
}
/// Linear probe from slot s whose key k0 was already loaded; UINT64_MAX when absent.
__device__ __forceinline__ uint64_t agg_lookup_from(const AggTableDev& t, uint64_t key, uint64_t s, uint64_t k0) {
  while (true) {
    if (k0 == key) return s;
    if (k0 == kEmptyKey) return ~0ULL;
    s = (s + 1) & t.mask;
    k0 = t.hot[s * t.hw];
  }
}
__device__ __forceinline__ uint64_t agg_lookup(const AggTableDev& t, uint64_t key) {
  if (key == kEmptyKey) return t.cold[(t.mask + 1) * t.cw] > 0 ? t.mask + 1 : ~0ULL;
  const uint64_t s = slot_of(key, t.shift);
  return agg_lookup_from(t, key, s, t.hot[s * t.hw]);
}

__device__ __forceinline__ bool local_bitmap_has(const LocalTableDev& t, uint64_t key) {
  const uint64_t d = key - static_cast<uint64_t>(t.bmin);
  return d < t.brange && ((__ldg(t.bitmap + (d >> 5)) >> (d & 31)) & 1u);
}
__device__ __forceinline__ uint64_t local_lookup(const LocalTableDev& t, uint64_t key) {
  if (t.bitmap) return local_bitmap_has(t, key) ? 0 : ~0ULL;  // no payload in bitmap mode
  if (key == kEmptyKey) return t.cnt[t.mask + 1] > 0 ? t.mask + 1 : ~0ULL;
  uint64_t s = slot_of(key, t.shift);
  while (true) {
    const uint64_t k = t.keys[s];
    if (k == key) return s;
    if (k == kEmptyKey) return ~0ULL;
    s = (s + 1) & t.mask;
  }
}
#endif

}  // namespace psg
