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

#include "device_common.cuh"

namespace psg {

// ---- launchers (defined in kernels.cu); all asynchronous on `stream` ----
/// d_tile_seg[t] = index of the segment holding tile t (tiles are scan_tile_rows() rows, never
/// spanning segments); built on the host next to the segment array.
void launch_scan(const ScanProgram& prog, const Segment* d_segs, const uint32_t* d_tile_seg, int nsegs,
                 uint64_t ntiles, void* stream);
int scan_tile_rows();  // rows per tile of k_scan

void launch_agg_init(const AggTableDev& t, uint64_t cap, void* stream);
void launch_bloom_build(const AggTableDev& t, uint64_t cap, void* stream);

// Local (CSR) table build from a materialised build batch.
void launch_local_init(uint64_t* keys, uint32_t* cnt, uint64_t cap, void* stream);
void launch_local_count(uint64_t* keys, uint32_t* cnt, uint64_t mask, int shift, const uint64_t* build_keys, uint64_t n,
                        unsigned int* max_cnt, void* stream);
void launch_local_fill(const uint64_t* keys, const uint32_t* start, uint32_t* cursor, uint64_t mask, int shift,
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
/// Key of a bit-packed row: min + (word >> shift & mask); mask == 0: the key column is the raw key.
struct KeyField {
  int64_t min;
  uint64_t mask;
  int32_t shift;
};
void launch_part_scatter(const uint64_t* const* in_cols, int ncols, uint64_t n, int key_col, int nparts,
                         const unsigned long long* dest_base, const unsigned long long* dest_cnt,
                         unsigned long long* cursor, uint64_t* send, void* stream, KeyField kf = KeyField{0, 0, 0});
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
// Dense finalisation (no sort): range + group count, key bitmap, popcounts, direct emit.
void launch_agg_range(const AggTableDev& t, uint64_t cap, unsigned long long* counter, void* stream);
void launch_agg_mark(const AggTableDev& t, uint64_t cap, uint64_t fmin, unsigned long long* bitmap, void* stream);
void launch_popc64(const unsigned long long* bitmap, uint64_t nwords, uint32_t* out, void* stream);
void launch_agg_emit_dense(const AggTableDev& t, uint64_t cap, uint64_t fmin, const unsigned long long* bitmap,
                           const uint32_t* prefix, int nc, const int32_t* col_kind, const int32_t* col_idx,
                           uint64_t* out_rows, void* stream);
size_t sort_pairs_i64(const uint64_t* keys_in, uint64_t* keys_out, const unsigned long long* v_in,
                      unsigned long long* v_out, uint64_t n, int end_bit, void* tmp, size_t tmp_bytes, void* stream);
size_t sort_pairs_u32(const uint32_t* keys_in, uint32_t* keys_out, const uint32_t* v_in, uint32_t* v_out, uint64_t n,
                      int end_bit, void* tmp, size_t tmp_bytes, void* stream);
void launch_gather64(const uint64_t* const* in_cols, int ncols, const uint64_t* idx, uint64_t n, uint64_t* const* out,
                     void* stream);
/// Phase-2 view of the bucketed aggregation (ScanProgram::bkt): nacc accumulator words per slot
/// (hot words 1..nacc); word[k] = the accumulator an unpacked probe sum k adds to.
struct BucketDev {
  const uint64_t* bkt;         // [nbuckets << sub_bits][cap]: sub-lists of a bucket (ScanProgram::bkt)
  const unsigned int* fill;
  uint32_t cap;
  int32_t sub_bits;
  int32_t nacc;
  int32_t shift[kMaxSums];
  uint64_t mask[kMaxSums];
  int64_t min[kMaxSums];
  int32_t word[kMaxSums];
  const uint64_t* ovf;            // {slot, entry} pairs of rows that found their bucket full
  const unsigned int* ovf_count;  // entries appended (may exceed ovf_cap: the engine re-runs)
  uint32_t ovf_cap;
};
/// One pass: fold each bucket, decoupled look-back for its output offset, rows in key order.
/// state: nbuckets words of scratch; *ticket receives the group total's inputs (see kernels.cu).
void launch_bucket_emit(const AggTableDev& t, const BucketDev& b, uint64_t nbuckets, uint64_t nslots,
                        unsigned long long* state, unsigned int* ticket, uint32_t* first_word, int nc,
                        const int32_t* col_kind, const int32_t* col_idx, uint64_t* out_rows, void* stream);
/// Own-key bitmap of a rank (N > 1) from the global one; cnt[0..1] += own / global popcounts.
void launch_own_mask(const unsigned long long* global, unsigned long long* own, uint64_t nwords, int64_t kmin, int nparts,
                     int self, unsigned long long* cnt, void* stream);
/// Every rank's local key bitmap (peer-mapped) and duplicate flag, for k_or_own.
struct OrPeers {
  const unsigned long long* bits[kMaxSlabPeers];
  const unsigned long long* rows[kMaxSlabPeers];  // rows that set bits (the build scan's kb_count)
  int32_t n;
};
/// Global (OR over ranks through NVLink) and own key bitmaps; cnt[0..3] += own bits, global bits,
/// |= overlap, += summed rows (k_or_own, kernels.cu).
void launch_or_own(const OrPeers& p, uint64_t nwords, int64_t kmin, int self, unsigned long long* global,
                   unsigned long long* own, unsigned long long* cnt, void* stream,
                   const unsigned long long* own_table = nullptr, uint32_t own_period = 0);
/// Ownership masks of one period of bitmap words (power-of-two node counts): partition_of(k) =
/// bits [13, 13 + log2 n) of k * kPartMul, which depend on k mod 2^(13 + log2 n) only, so word w's
/// owned-bit mask is table[w mod P], P = own_period(n) words. 0: no period (n not a power of two).
uint32_t own_period(int nparts);
void launch_own_table(int64_t kmin, int nparts, int self, unsigned long long* table, void* stream);
/// Device-side barrier over the symmetric heap (N > 1): flag[p] is peer p's flag array (one word
/// per source rank), own this rank's. Each rank stores the epoch into every peer's slot for it
/// (release, system scope), then waits until every slot of its own array holds the epoch
/// (acquire); a rank missing for ~10 s sets *err instead of hanging the GPU.
struct PeerFlags {
  uint32_t* flag[kMaxSlabPeers];
};
void launch_peer_barrier(const PeerFlags& f, const uint32_t* own, int self, int n, uint32_t epoch, unsigned int* err,
                         void* stream);
/// Small host reads gathered into one launch: word i = *src[i] (a u32 when bit i of w32 is set)
/// stored into mapped pinned host memory, so a batch of scalars costs one kernel and one stream
/// sync instead of one pageable D2H copy (each a host round trip with the GPU idle) per value.
struct GatherWords {
  const void* src[24];
  uint32_t w32;
  int32_t n;
};
void launch_gather_words(const GatherWords& g, unsigned long long* host_mapped, void* stream);
/// Bulk L2 prefetch of [p, p + bytes) (16-byte aligned).
void launch_l2_prefetch(const void* p, uint64_t bytes, void* stream);
/// Peer-slab shuffle, owner side (kernels.cu k_slab_consume).
struct SlabConsume {
  const uint64_t* src_rows[kMaxSlabPeers];             // rows source r holds for this rank (peer-mapped outbox, or the local inbox)
  const unsigned long long* src_cnt[kMaxSlabPeers];    // rows source r stored here (peer-mapped; null: none)
  uint64_t cap;                                        // rows per region
  int32_t nsrc;
  int32_t npack;                                       // packed fields: key, then the probe sums
  int32_t pshift[kMaxSums + 1];
  uint64_t pmask[kMaxSums + 1];
  int64_t pmin[kMaxSums + 1];
  // the bucket entry format of the probe kernel (ScanProgram::bkt_*)
  uint64_t* bkt;
  unsigned int* fill;
  uint32_t bcap;
  int32_t bsub_bits;
  int32_t bshift[kMaxSums];
  uint64_t bmask[kMaxSums];
  int64_t bmin[kMaxSums];
  uint64_t* ovf;
  unsigned int* ovf_count;
  uint32_t ovf_cap;
  unsigned long long* received;                        // += rows consumed (stats)
  int32_t diag;                                        // PSG_SLAB_DIAG (measurement only)
};
void launch_slab_consume(const AggTableDev& t, const SlabConsume& c, void* stream);
/// Rank records of a key bitmap in two launches (replaces popc64 + scan + krec_build): per-tile
/// popcounts into tile_sums (rank_tiles(n) words), then krank[w] = the popcount of words < w and
/// krec[w] = {bits[w], krank[w]} (the bitmap tile is re-read from L2).
uint64_t rank_tiles(uint64_t n);
void launch_rank_records(const unsigned long long* bits, uint64_t n, uint32_t* tile_sums, uint32_t* krank,
                         unsigned long long* krec, void* stream);
void launch_krec_build(const unsigned long long* bits, const uint32_t* krank, uint64_t n, unsigned long long* krec,
                       void* stream);
void launch_part_hist(const uint64_t* keys, uint64_t n, int nparts, unsigned long long* counts, void* stream);
void launch_minmax_i64(const uint64_t* keys, uint64_t n, long long* out, void* stream);
void launch_bitmap_set(const uint64_t* keys, uint64_t n, int64_t bmin, uint32_t* bitmap, unsigned int* dup, void* stream);
struct RankSums {
  const uint64_t* col[kMaxSums];
};
void launch_rank_build(const AggTableDev& t, const uint64_t* keys, const RankSums& bs, uint64_t n, bool first,
                       bool write_hot, void* stream);
void launch_bloom_keys(const uint64_t* keys, uint64_t n, uint32_t* bloom, int shift, void* stream);
void launch_iota_u32(uint32_t* out, uint64_t n, void* stream);
void launch_rows_from_cols(const uint64_t* const* cols, int ncols, uint64_t n, uint64_t* out_rows, void* stream);

// Block-codec inflate (inflate.cu): one zlib stream per job, decoded in HBM.
struct InflateJob {
  const uint8_t* src;  // compressed stream (4-byte aligned; may be read up to 3 bytes past csize)
  uint8_t* dst;        // output (8-byte aligned), exactly usize bytes on success
  uint32_t csize, usize;
};
/// Decodes every job; sets *d_err to nonzero if any stream is invalid (zlib's Z_DATA_ERROR,
/// size mismatch or Adler-32 mismatch).
void launch_inflate(const InflateJob* d_jobs, uint32_t njobs, unsigned int* d_err, void* stream);

uint64_t kernel_launch_count();
void count_external_launch();

}  // namespace psg
