/*
 * psg.h — C-ABI boundary of the B200-native PystachIO hot path (paper 2512.02862).
 *
 * Plain pointers and sizes only; no torch/CUDA types cross this boundary. Every entry point
 * replaces one reference interface (cited as /root/reference/proj/... file:line) so a maintainer
 * can bind it from the reference's own C++  or from Python via ctypes
 * (paper_2512_02862_b200/__init__.py).
 *
 * Threading: one host control thread per GPU owns a psg_ctx and issues every call for it
 * (mirrors the reference's one-control-thread-per-node rule, socket_fabric.hpp:48-49).
 * Errors: every int-returning call returns PSG_OK (0) or a psg_status code mapped 1:1 onto the
 * reference's exception classes (errors.hpp:21-87); psg_last_error() gives the message
 * (thread-local).
 */
#ifndef PSG_H_
#define PSG_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PSG_ABI_VERSION 2

/* Status codes — 1:1 with pystachio::Error subclasses (errors.hpp:21-87) + CUDA/NCCL. */
typedef enum psg_status {
  PSG_OK = 0,
  PSG_ERR_UNKNOWN_COLUMN = 1,        /* UnknownColumn            errors.hpp:26-29 */
  PSG_ERR_MEMORY_EXCEEDED = 2,       /* MemoryExceeded           errors.hpp:31-37 */
  PSG_ERR_STREAM_CLOSED = 3,         /* StreamClosed             errors.hpp:39-42 */
  PSG_ERR_IO_FAILURE = 4,            /* IoFailure                errors.hpp:44-47 */
  PSG_ERR_CORRUPT_FOOTER = 5,        /* CorruptFooter            errors.hpp:49-52 */
  PSG_ERR_COLLECTIVE_ORDER = 6,      /* CollectiveOrderViolation errors.hpp:54-58 */
  PSG_ERR_PEER_DISCONNECTED = 7,     /* PeerDisconnected         errors.hpp:60-63 */
  PSG_ERR_CHECKSUM_MISMATCH = 8,     /* ChecksumMismatch         errors.hpp:65-68 */
  PSG_ERR_INVALID_INPUT = 9,         /* InvalidInput             errors.hpp:70-73 */
  PSG_ERR_INFEASIBLE_BUDGET = 10,    /* InfeasibleBudget         errors.hpp:75-78 */
  PSG_ERR_MALFORMED_TRACE = 11,      /* MalformedTrace           errors.hpp:80-83 */
  PSG_ERR_EMPTY_TRACE = 12,          /* EmptyTrace               errors.hpp:84-87 */
  PSG_ERR_CUDA = 100,                /* CUDA runtime failure (no CPU fallback exists) */
  PSG_ERR_NCCL = 101,                /* NCCL failure */
  PSG_ERR_INTERNAL = 102
} psg_status;

/* LogicalType (types.hpp:29): both 8-byte words. */
#define PSG_INT64 0
#define PSG_FLOAT64 1

/* ExecMode (pipeline.hpp:124). All four return identical result multisets. */
#define PSG_MODE_BLOCKING 0   /* FullyBlocking: ingest everything, then compute   */
#define PSG_MODE_FASTIO 1     /* FastIO: per-chunk waves, phase-sequential         */
#define PSG_MODE_COMBINED 2   /* Combined: both scans share the ingest pool         */
#define PSG_MODE_OVERLAPPED 3 /* Overlapped: ingest/shuffle/compute overlap chunk by chunk */

/* Codec (psto.hpp:30). */
#define PSG_CODEC_IDENTITY 0
#define PSG_CODEC_BLOCK 1

typedef struct psg_ctx psg_ctx;
typedef struct psg_result psg_result;
typedef struct psg_staged psg_staged;

/* A host columnar batch (ChunkBatch, types.hpp:101-156): ncols columns of nrows raw 8-byte words. */
typedef struct psg_batch {
  uint32_t ncols;
  uint64_t nrows;
  const char* const* names; /* ncols column names */
  const uint8_t* types;     /* ncols PSG_INT64 / PSG_FLOAT64 */
  uint64_t* const* cols;    /* ncols host pointers to nrows words each */
} psg_batch;

/* A predicate atom (PredicateAtom, predicate.hpp:30-41). op: "<","<=","==","!=",">=",">". */
typedef struct psg_atom {
  const char* column;
  const char* op;
  int literal_is_float; /* 0: literal_i, 1: literal_f (std::variant<int64_t,double>) */
  int64_t literal_i;
  double literal_f;
} psg_atom;

/* Per-query statistics (PipelineResult, pipeline.hpp:138-149, plus device-side timings). */
typedef struct psg_stats {
  double runtime_s;            /* end - start on this rank (host wall, around the whole call) */
  double storage_phase_s;      /* phased modes: ingest phase */
  double network_phase_s;      /* phased modes: shuffle phase */
  uint64_t peak_bytes;         /* peak device bytes from the engine pool */
  uint64_t bytes_received;     /* shuffle payload bytes received from peers */
  uint64_t ingest_bytes;       /* file bytes moved host->HBM */
  uint64_t result_bytes;       /* result bytes moved HBM->host */
  uint64_t kernel_launches;    /* our kernels launched by this call */
  uint64_t waves;              /* shuffle waves */
  double probe_kernel_ms;      /* summed CUDA-event time of the dominant fused probe kernel */
  uint64_t probe_kernel_launches;
  uint64_t probe_kernel_bytes; /* algorithmic bytes (input column chunks) those launches scanned */
  double device_ms;            /* CUDA-event time on the engine's compute stream, first to last op */
  uint64_t result_rows;        /* rows of this rank's result (also when rows stay on the device) */
  double io_wait_s;            /* host time the control thread waited for storage reads */
  uint64_t jit_compiles;       /* NVRTC kernel compilations during this call (cached afterwards) */
  uint64_t h2d_bytes;          /* host->HBM bytes copied (compressed for block-codec chunks) */
  uint64_t agg_table;          /* shuffle-join table kind: 0 none (no aggregate), 1 hashed, 2 hashed +
                                  Bloom screen, 3 hashed + exact key bitmap, 4 rank-indexed (dense
                                  unique build keys), 5 symmetric peer-mapped (fused NVLink) */
  uint64_t bytes_sent;         /* shuffle payload bytes sent to peers */
  double exchange_ms;          /* summed CUDA-event time of the shuffle send/recv groups */
  uint64_t bucket_overflow;    /* rows that found their aggregation bucket full (bucketed aggregation) */
  uint64_t shuffle_fused;      /* 1: the shuffle ran inside the probe kernel (peer-slab stores over
                                  NVLink; bytes_received counts them, exchange_ms stays 0) */
} psg_stats;

/* ---- library ---- */
int psg_abi_version(void);
const char* psg_last_error(void);

/* Host-only shuffle protocol (the functions every rank evaluates on all-gathered / all-reduced
 * inputs; run_waves size exchange, pipeline.cpp:690-722):
 *  psg_shuffle_plan: from the n x n count matrix [src][dst] (row-major), rank me's send offsets
 *    into its destination-major slab and receive offsets per source (rows).
 *  psg_pack_plan: one-word row layout from all-reduced per-column bounds (column 0 = key); fits=0
 *    when the fields do not fit in 64 bits.
 *  psg_partition_of: partition_of(key) = ((key * 0x9E3779B97F4A7C15) >> 13) % nparts
 *    (hashing.hpp:35-37), the destination of a shuffled row. */
int psg_shuffle_plan(const uint64_t* matrix, int n, int me, uint64_t* send_off, uint64_t* recv_off,
                     uint64_t* send_rows, uint64_t* recv_rows);
int psg_pack_plan(const int64_t* lo, const int64_t* hi, int ncols, int64_t* min, int* shift, uint64_t* mask,
                  int* fits);
int psg_partition_of(const int64_t* keys, uint64_t n, uint32_t nparts, uint32_t* out);

/* ---- distributed-join microbenchmark (run_join / run_sim_join, join.cpp:55-124, join_harness.cpp:43-97) ----
 * The symmetric-repartitioning hash join in the reference's four schedules on CUDA streams:
 * variant 0 blocking (whole tables, one stream, a cudaMalloc per buffer), 1 blocking-opt (pooled),
 * 2 chunking, 3 deferred (the probe of wave w is issued after wave w+k's shuffle). */
typedef struct psg_join_spec {
  int variant;           /* JoinVariant (join.hpp:31) */
  int stream_count;      /* compute streams of the chunked variants (join.hpp:42) */
  uint64_t chunk_rows;   /* wave size (join.hpp:40) */
} psg_join_spec;
typedef struct psg_join_workload { /* SyntheticJoinSpec (workload.hpp:27-33) */
  uint64_t build_rows, probe_rows;
  int payload_cols;
  double hit_ratio;
  uint64_t seed;
} psg_join_workload;
typedef struct psg_join_stats {
  double runtime_s;       /* host wall time of the join (inputs in host memory, H2D included) */
  double device_ms;       /* CUDA-event time, first to last step */
  uint64_t result_rows;   /* this rank's joined rows */
  uint64_t bytes_received;/* shuffle payload bytes from peers */
  uint64_t left_waves, right_waves;
  uint64_t host_syncs;    /* data-dependent waits of the control thread */
} psg_join_stats;
/* Host-only: the schedule (PlanStep list, join.hpp:70-95) as triples {phase, stream, wave};
 * phases in PlanStep::Phase order (concat_left=0 ... drain=10). */
int psg_join_schedule(int variant, int stream_count, int left_waves, int right_waves, int32_t* out, size_t cap_steps,
                      size_t* nsteps);
/* Runs this rank's part of the join over its slice (slice_for_node) of the synthetic workload;
 * rows (optional, collect) = build payload ++ probe columns per joined row. */
int psg_run_synthetic_join(psg_ctx* ctx, const psg_join_spec* spec, const psg_join_workload* workload, int collect_rows,
                           psg_join_stats* stats, psg_result** rows);

/* Host-only: parses + validates a plan like QueryPlan::from_json_text (pipeline.cpp:108-156,
 * validate :178-196) for node `node` of `nodes` and writes the resolved scans as JSON
 * {"scans":[{"table","replicated","paths":[...]}],"shuffle":id|null} into out (NUL-terminated,
 * truncated to cap; *needed = full size + 1). Errors: InvalidInput (bad JSON / plan shape),
 * IoFailure (a path matches no file). */
int psg_plan_resolve(const char* plan_json, const char* data_root, int node, int nodes, char* out, size_t cap,
                     size_t* needed);

/* ---- per-GPU context (ExecEnv + Fabric + DeviceManager + MetadataCache, exec.hpp:84-92) ---- */
/* device: CUDA ordinal; rank/nranks: this GPU's node id and the node count (Fabric::node_count). */
int psg_ctx_create(int device, int rank, int nranks, psg_ctx** out);
/* NCCL plumbing for nranks > 1 (replaces SocketFabric, socket_fabric.hpp:50-118): rank 0 makes
 * the 128-byte id, the host transport (torch.distributed) broadcasts it, every rank inits. */
int psg_comm_unique_id(void* out128);
int psg_ctx_init_comm(psg_ctx* ctx, const void* id128);
/* Engine knobs: io_threads (0 = plan.io_workers), batch bytes per ingest slot, pinned slots. */
int psg_ctx_set_ingest(psg_ctx* ctx, int io_threads, uint64_t batch_bytes, int pinned_slots);
/* Semi-join (Bloom) pre-filter of the shuffled probe side: 1 = on (default), 0 = off. */
int psg_ctx_set_semijoin(psg_ctx* ctx, int enabled);
/* Fused NVLink shuffle for grouped aggregates (nranks > 1): build inserts and probe+aggregate go
 * straight into the owner rank's hash table through CUDA-IPC-mapped peer memory (system-scope
 * atomics), replacing partition -> count exchange -> ncclSend/Recv -> consume. Collective on the
 * first enable (maps every peer's symmetric heap, PSG_SYMM_MB, default 4096). 0 (default) = the
 * NCCL path, which measured faster for Q3 (remote atomics cost NVLink bandwidth). */
int psg_ctx_set_fused_shuffle(psg_ctx* ctx, int enabled);
void psg_ctx_destroy(psg_ctx* ctx);

/* ---- plan execution: execute_plan (pipeline.hpp:153-155, pipeline.cpp:924-929) ----
 * plan_json is the reference's plan JSON (QueryPlan::from_json_text, pipeline.cpp:108-156);
 * {data}/{node}/{nodes} are substituted with data_root / ctx rank / ctx nranks.
 * Storage-resident: reads PSTO files, streams chunks into HBM on copy streams, runs the fused
 * kernels, shuffles over NCCL when nranks > 1, returns this rank's rows. */
int psg_execute_plan(psg_ctx* ctx, const char* plan_json, const char* data_root, int mode,
                     psg_result** out);

/* Extension (the Q6 analog): plans WITHOUT a shuffled join - one root stream
 * (a scan, or a chain of local joins against replicated scans) ending in a global aggregate -
 * which the reference's execute_plan rejects (pipeline.cpp:334-335; psg_execute_plan keeps that
 * InvalidInput). No exchange: each rank returns its node's unmerged partial row [rows, sums...]
 * (the global-aggregate semantics of pipeline.cpp:277-281). */
/* Measurement: moves every column chunk the plan reads storage -> pinned -> HBM through the same
 * ingest session psg_execute_plan uses (same I/O threads, ring and copy stream; block-codec
 * chunks are also inflated) and runs no query kernels. stats: runtime_s, h2d_bytes,
 * ingest_bytes, io_wait_s - the ingest term of the end-to-end roofline (bench.cpp:35-40 t_min). */
int psg_ingest_probe(psg_ctx* ctx, const char* plan_json, const char* data_root, psg_stats* out);

int psg_execute_local(psg_ctx* ctx, const char* plan_json, const char* data_root, int mode,
                      psg_result** out);

/* HBM-resident variant: psg_stage_plan reads every file the plan touches into HBM once;
 * psg_execute_staged runs the query over the staged bytes (no host I/O). When out is NULL the
 * result stays on the device (its row count is still available through stats). */
int psg_stage_plan(psg_ctx* ctx, const char* plan_json, const char* data_root, psg_staged** out);
int psg_execute_staged(psg_ctx* ctx, psg_staged* staged, int mode, psg_result** out,
                       psg_stats* stats);
void psg_staged_free(psg_staged* staged);

/* ---- results (PipelineResult rows/schema, pipeline.hpp:138-149) ---- */
int psg_result_shape(const psg_result* r, uint64_t* nrows, uint32_t* ncols);
int psg_result_field(const psg_result* r, uint32_t col, const char** name, int* type);
const uint64_t* psg_result_data(const psg_result* r); /* row-major nrows*ncols words */
int psg_result_stats(const psg_result* r, psg_stats* out);
/* Result checksum (host-side, over the rows already on the host): rowhash = sum over rows of
 * FNV-1a64 of the row's little-endian words mod 2^64 (additive over ranks, independent of row
 * order) and per-column wrap-around sums into colsums[0..min(ncols, ncols_cap)). */
int psg_result_checksum(const psg_result* r, uint64_t* rowhash, uint64_t* colsums, uint32_t ncols_cap);
void psg_result_free(psg_result* r);

/* ---- operator adapters (ops.hpp:35-83): host batch -> HBM -> kernel -> host ---- */
/* filter (ops.cpp:45-54): order-preserving. */
int psg_filter(psg_ctx* ctx, const psg_batch* in, const psg_atom* atoms, uint32_t natoms,
               psg_result** out);
/* partition (ops.cpp:56-78): h(key) % nparts, order-preserving within each part.
 * hash_kind: 0 = MultiplyShift, 1 = Identity (hashing.hpp:22). Output rows are grouped by part;
 * part_rows receives nparts counts. */
int psg_partition(psg_ctx* ctx, const psg_batch* in, const char* key_column, uint32_t nparts,
                  int hash_kind, psg_result** out, uint64_t* part_rows);
/* HashTable::build + probe (ops.cpp:105-222): inner join, output = build payload ++ probe
 * columns ("_p" suffix on name clash). Row order unspecified (the reference's tests compare
 * multisets). */
int psg_hash_join(psg_ctx* ctx, const psg_batch* build, const char* build_key,
                  const psg_batch* probe, const char* probe_key, psg_result** out);

/* codec_decompress (psto.cpp:133-143), batched and on the GPU: n chunks, host buffers.
 * codec 0 = identity (copies src to dst; needs src_len == dst_len), 1 = block (zlib stream ->
 * exactly dst_len bytes). Any invalid stream or size mismatch -> PSG_ERR_IO_FAILURE
 * ("inflate failed"), like the reference. */
int psg_codec_decompress(psg_ctx* ctx, int codec, uint64_t n, const void* const* src, const uint64_t* src_len,
                         void* const* dst, const uint64_t* dst_len);

/* HashTable (ops.hpp:49-82) as a GPU handle: build over nbatches batches of one schema
 * (duplicates keep every row; hash_kind as in psg_partition, accepted for API parity), then
 * any number of lookups / probes. The materialised build side is the concatenation of the
 * batches (row r = r-th row overall). Free every table before its context. */
typedef struct psg_hashtable psg_hashtable;
int psg_hashtable_build(psg_ctx* ctx, const psg_batch* batches, uint32_t nbatches, const char* key_column,
                        int hash_kind, psg_hashtable** out);
/* row_count() and the number of payload columns (build columns minus the key). */
int psg_hashtable_shape(const psg_hashtable* t, uint64_t* rows, uint32_t* payload_cols);
/* key_at(row) / payload_at(col, row) for every payload column (build order, key skipped). */
int psg_hashtable_row(const psg_hashtable* t, const char* key_column, uint64_t row, int64_t* key,
                      uint64_t* payload);
/* lookup(key) for n keys at once: offsets[0..n] (CSR) into rows_out, the build-row indices that
 * carry each key (a multiset per key, like the reference's chained buckets); *total = matches.
 * InvalidInput when total > cap (offsets and *total are still filled). */
int psg_hashtable_lookup(psg_ctx* ctx, const psg_hashtable* t, const int64_t* keys, uint64_t n,
                         uint64_t* offsets, uint64_t* rows_out, uint64_t cap, uint64_t* total);
/* probe (ops.cpp:173-222): build payload ++ probe columns ("_p" on a name clash). */
int psg_hashtable_probe(psg_ctx* ctx, const psg_hashtable* t, const psg_batch* probe, const char* probe_key,
                        psg_result** out);
void psg_hashtable_free(psg_hashtable* t);
/* concat (ops.cpp:80-98): batches of one schema into one (InvalidInput on a schema mismatch). */
int psg_concat(psg_ctx* ctx, const psg_batch* batches, uint32_t nbatches, psg_result** out);

/* ---- PSTO format (psto.hpp) ---- */
/* TableWriter (psto.cpp:144-229): writes a batch as a PSTO file. Returns row groups written. */
int psg_psto_write(const char* path, const psg_batch* batch, uint64_t row_group_rows, int codec,
                   uint64_t* groups_written);
/* parse_footer_file (psto.cpp:294-318): rows, columns, row groups, codec. */
int psg_psto_inspect(const char* path, uint64_t* rows, uint32_t* ncols, uint64_t* groups,
                     int* codec);

/* ---- workload generator: gen_workload(kind=tpch) (bench.cpp:85-114) ----
 * Byte-identical to the reference generator (pinned by tests/golden/gen_hashes.json). */
int psg_gen_tpch(const char* out_dir, double scale, int nodes, int devices, uint64_t seed,
                 int codec, uint64_t row_group_bytes, int threads);

/* gen_workload(kind = synthetic join) (bench.cpp:93-99, workload.cpp:27-71): build table
 * {bk, bp0..} with keys 0..build_rows-1 shuffled, probe table {pk, pp0..} with hit_ratio of its
 * keys in the build range; round-robin node shards dev{(k + i) % devices}/{build,probe}.node{k}.psto
 * and manifest.json. Reference defaults: 120000, 320000, 3, 0.5. Byte-identical to the reference. */
int psg_gen_synthetic(const char* out_dir, int nodes, int devices, uint64_t seed, int codec,
                      uint64_t row_group_bytes, uint64_t build_rows, uint64_t probe_rows, int payload_cols,
                      double hit_ratio);

/* ---- query compiler self-test: NVRTC-compiles representative fused-scan programs for sm_100a
 * (no GPU needed). Returns the number of failing programs (0 = ok), -1 on error; log gets NVRTC
 * output for failures. */
int psg_jit_selftest(char* log, size_t cap);

/* ---- Eq. 1 roofline: t_min (bench.cpp:35-40) ---- */
double psg_tmin(uint64_t ssd_read_size_agg, double ssd_read_bw_agg, uint64_t net_recv_size_node,
                double net_bw);

#ifdef __cplusplus
}
#endif
#endif /* PSG_H_ */
