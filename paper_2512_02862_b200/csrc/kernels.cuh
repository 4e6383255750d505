// Device-side data structures and kernel launchers of the fused scan pipeline.
//
// One generic fused kernel (k_scan) runs the per-chunk hot loop of the reference's scan path
// (decode_group -> filter -> transform/apply_chain, scan.cpp:190-268, pipeline.cpp:431-448) and
// ends in one of four sinks, which replace the reference's downstream operators:
//   SINK_MATERIALIZE : order-preserving-per-tile stream compaction of the needed columns
//                      (filter/gather ops.cpp:29-54; partition input; DynamicBuffer concat)
//                      + optional per-destination histogram (partition ops.cpp:56-78)
//   SINK_BUILD       : insert into the shuffle-join aggregation table (HashTable::build
//                      ops.cpp:105-159 specialised for group-by == join key)
//   SINK_PROBE       : probe + grouped aggregation in the table slot (HashTable::probe
//                      ops.cpp:173-222 -> deliver -> HashAggregator::add pipeline.cpp:275-294)
//   SINK_PROBE_GLOBAL: probe + global aggregate (one row per node, pipeline.cpp:277-281)
// The kernel interprets a small runtime "program" (predicate atoms, a chain of unique-key local
// joins, register map), so any plan of the reference's shape runs through the same code.
#pragma once

#include <cstdint>

namespace psg {

constexpr uint64_t kEmptyKey = 0x8000000000000000ULL;  // INT64_MIN; real INT64_MIN keys use the spill slot
constexpr int kMaxIn = 16;
constexpr int kMaxAtoms = 8;
constexpr int kMaxJoins = 4;
constexpr int kMaxPayload = 8;
constexpr int kMaxRegs = 26;  // dynamic smem = n_regs * 4 rows * 256 threads * 8 B <= 208 KiB
constexpr int kMaxOut = 16;
constexpr int kMaxSums = 8;
constexpr int kMaxParts = 64;
constexpr int kBlock = 256;

enum SinkKind : int { SINK_MATERIALIZE = 0, SINK_BUILD = 1, SINK_PROBE = 2, SINK_PROBE_GLOBAL = 3, SINK_COUNT = 4 };

/// One row group (or one received/materialised run): rows + a device pointer per input column.
struct Segment {
  const uint64_t* col[kMaxIn];
  uint64_t rows;
  uint64_t tile_begin;  // first tile index of this segment (prefix over segments)
};

struct AtomDesc {
  int32_t reg;
  int32_t op;        // CmpOp
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
  int32_t pad;
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
  unsigned long long* global_acc;       // SINK_PROBE_GLOBAL: [rows, probe sums..., build sums...]
  int32_t global_float[2 * kMaxSums + 1];
};

// ---- launchers (defined in kernels.cu); all asynchronous on `stream` ----
void launch_scan(const ScanProgram& prog, const Segment* d_segs, int nsegs, uint64_t ntiles, int tile_rows_log2,
                 void* stream);
int scan_tile_rows();  // rows per tile of k_scan

void launch_agg_init(const AggTableDev& t, uint64_t cap, void* stream);
void launch_bloom_build(const AggTableDev& t, uint64_t cap, void* stream);

// Local (CSR) table build from a materialised build batch.
void launch_local_init(uint64_t* keys, uint32_t* cnt, uint64_t cap, void* stream);
void launch_local_count(uint64_t* keys, uint32_t* cnt, uint64_t mask, const uint64_t* build_keys, uint64_t n,
                        unsigned int* max_cnt, void* stream);
void launch_local_fill(const uint64_t* keys, const uint32_t* start, uint32_t* cursor, uint64_t mask,
                       const uint64_t* build_keys, const uint64_t* const* src_cols, uint64_t* const* dst_cols,
                       int ncols, uint64_t n, void* stream);
/// Exclusive scan of n u32 -> u32 (CUB), temp managed by caller-provided scratch (size query when tmp==nullptr).
size_t exclusive_scan_u32(const uint32_t* in, uint32_t* out, uint64_t n, void* tmp, size_t tmp_bytes, void* stream);
size_t exclusive_scan_u64(const unsigned long long* in, unsigned long long* out, uint64_t n, void* tmp,
                          size_t tmp_bytes, void* stream);

// Generic join with duplicates (probe_expand): pass 1 counts, pass 2 writes.
void launch_expand_count(LocalTableDev t, const uint64_t* probe_keys, uint64_t n, uint32_t* counts, void* stream);
void launch_expand_write(LocalTableDev t, const uint64_t* probe_keys, uint64_t n, const uint32_t* offsets,
                         const uint64_t* const* probe_cols, int nprobe, uint64_t* const* out_cols, void* stream);

// Partition scatter (pipeline shuffle): rows of a materialised batch into dest-major send regions.
void launch_part_scatter(const uint64_t* const* in_cols, int ncols, uint64_t n, int key_col, int nparts,
                         const unsigned long long* dest_base, const unsigned long long* dest_cnt,
                         unsigned long long* cursor, uint64_t* send, void* stream);
// Stable partition for the op-level API: dest id per row.
void launch_part_ids(const uint64_t* keys, uint64_t n, int nparts, int identity, uint32_t* ids, void* stream);
void launch_gather(const uint64_t* const* in_cols, int ncols, const uint32_t* idx, uint64_t n, uint64_t* const* out,
                   void* stream);

// Grouped-result finalisation: compact occupied slots with hits > 0 into rows, sort by signed key.
void launch_agg_compact(const AggTableDev& t, uint64_t cap, uint64_t* out_keys, unsigned long long* out_slots,
                        unsigned long long* counter, void* stream);
void launch_agg_emit(const AggTableDev& t, const uint64_t* sorted_keys, const unsigned long long* sorted_slots,
                     uint64_t n, int ncols_out, const int32_t* col_kind, const int32_t* col_idx, uint64_t* out_rows,
                     void* stream);
size_t sort_pairs_i64(const uint64_t* keys_in, uint64_t* keys_out, const unsigned long long* v_in,
                      unsigned long long* v_out, uint64_t n, void* tmp, size_t tmp_bytes, void* stream);
size_t sort_pairs_u32(const uint32_t* keys_in, uint32_t* keys_out, const uint32_t* v_in, uint32_t* v_out, uint64_t n,
                      int end_bit, void* tmp, size_t tmp_bytes, void* stream);
void launch_iota_u32(uint32_t* out, uint64_t n, void* stream);
void launch_rows_from_cols(const uint64_t* const* cols, int ncols, uint64_t n, uint64_t* out_rows, void* stream);

uint64_t kernel_launch_count();

}  // namespace psg
