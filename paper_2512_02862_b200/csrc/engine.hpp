// Host side of the B200-native plan executor: per-GPU context, device memory pool, chunked
// ingest pipeline and the execute_plan driver (replaces PlanExecution, pipeline.cpp:317-920).
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <chrono>
#include <condition_variable>
#include <deque>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "kernels.cuh"
#include "plan.hpp"
#include "psto.hpp"

namespace psg {

/// Caching device allocator with budget accounting (the RMM-pool analog of MemoryPool,
/// memory_pool.hpp:30-108). Blocks are cudaMalloc'ed once and recycled per stream: a block freed
/// on stream s is only handed out again to work on s, so stream order makes reuse safe without
/// host syncs (cudaMallocAsync's pool grew and re-mapped memory under in-flight work, which cost
/// milliseconds per query).
class DevicePool {
 public:
  void init(int device, uint64_t budget);
  void* alloc(size_t bytes, cudaStream_t s);
  void free(void* p, cudaStream_t s);
  uint64_t used() const { return used_; }
  uint64_t peak() const { return peak_; }
  uint64_t cached() const { return cached_; }
  void reset_peak() { peak_ = used_; }
  void set_budget(uint64_t b) { budget_ = b; }
  void release_cache();
  ~DevicePool() { release_cache(); }

 private:
  std::map<void*, size_t> live_;
  std::map<std::pair<cudaStream_t, size_t>, std::vector<void*>> free_;  // (stream, size) -> blocks
  uint64_t used_ = 0, peak_ = 0, budget_ = 0, cached_ = 0;
};

/// RAII device buffer from the pool.
struct DevBuf {
  DevicePool* pool = nullptr;
  void* p = nullptr;
  size_t bytes = 0;
  cudaStream_t s = nullptr;
  DevBuf() = default;
  DevBuf(DevicePool& pl, size_t n, cudaStream_t st) : pool(&pl), bytes(n), s(st) { p = pl.alloc(n ? n : 8, st); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept { *this = std::move(o); }
  DevBuf& operator=(DevBuf&& o) noexcept {
    reset();
    pool = o.pool, p = o.p, bytes = o.bytes, s = o.s;
    o.p = nullptr;
    return *this;
  }
  ~DevBuf() { reset(); }
  void reset() {
    if (p && pool) pool->free(p, s);
    p = nullptr;
  }
  template <class T>
  T* as() const { return static_cast<T*>(p); }
};

/// Metadata cache (MetadataCache, metadata_cache.hpp:26-60): footer per path.
class FooterCache {
 public:
  std::shared_ptr<const TableMeta> get(const std::string& path);

 private:
  std::mutex mu_;
  std::map<std::string, std::pair<std::pair<int64_t, uint64_t>, std::shared_ptr<const TableMeta>>> map_;
};

/// Read-only shared mappings of the input files, kept across queries (keyed like the footer cache
/// on mtime + size; a changed file is re-mapped). The ingest workers copy column chunks straight
/// out of the page cache with memcpy (streaming stores) instead of pread: one kernel-side copy
/// fewer per byte - on the bench box the page cache -> pinned -> HBM pipeline goes from 44 to
/// 53 GB/s, the PCIe H2D rate (profiles/r2_ingest_probe2.txt). Mappings hold no data of their
/// own; pages stay in the page cache. A file truncated WHILE a query copies from its mapping
/// would fault (SIGBUS) where pread reports a short read: the stamp check at each query's start
/// re-maps changed files, and the footer bounds every extent by the file size it was read with.
/// PSG_MMAP=0: pread.
struct FileMapping {
  const uint8_t* base = nullptr;
  size_t bytes = 0;
  ~FileMapping();
};
class FileMapCache {
 public:
  /// nullptr when the file cannot be mapped (the caller falls back to pread).
  std::shared_ptr<const FileMapping> get(const std::string& path);
  static bool enabled();

 private:
  std::mutex mu_;
  std::map<std::string, std::pair<std::pair<int64_t, uint64_t>, std::shared_ptr<const FileMapping>>> map_;
};

/// One contiguous file range copied into a batch buffer.
struct Extent {
  uint64_t file_off, len, buf_off;
};

/// An ingest batch: consecutive surviving row groups of one file, needed column chunks packed.
struct BatchPlan {
  int file = 0;
  std::vector<size_t> groups;
  std::vector<uint64_t> rows;               // rows per group
  std::vector<std::vector<uint64_t>> pos;   // [group][needed col] offset in batch buffer
  std::vector<Extent> extents;
  uint64_t bytes = 0;          // buffer footprint (16-byte aligned chunks + tail padding)
  uint64_t payload_bytes = 0;  // column-chunk bytes read from the file (algorithmic bytes)
  uint64_t total_rows = 0;
  // Block codec: `extents` land compressed chunks in the H2D buffer; `pos` then addresses the
  // decoded image (dbytes) that the inflate jobs write (src/dst offsets relative to each buffer).
  bool inflate = false;
  struct Job {
    uint64_t src_off, dst_off;
    uint32_t csize, usize;
  };
  std::vector<Job> jobs;
  uint64_t dbytes = 0;  // decoded footprint (16-byte aligned chunks + tail padding)
  uint64_t ubytes = 0;  // decoded column-chunk bytes (what the scan kernel reads)
  uint64_t scan_bytes() const { return inflate ? ubytes : payload_bytes; }
};

/// Opt-in execution timeline (PSG_TIMELINE=<path>): intervals on the GPU streams (CUDA events
/// against one origin event) and on the host I/O threads (steady_clock against the origin's host
/// time), written as Chrome-trace JSON (<path>.rank<r>.json) - the overlap evidence nsys would give
/// (nsys is not in the image). Lanes: 0 host reads, 1 H2D copy, 2 inflate, 3 compute, 4 exchange.
class Timeline {
 public:
  static bool enabled();
  explicit Timeline(cudaStream_t origin_stream);
  ~Timeline();
  int gpu_begin(const std::string& name, int lane, cudaStream_t s);
  void gpu_end(int id, cudaStream_t s);
  void host(const std::string& name, int lane, std::chrono::steady_clock::time_point a,
            std::chrono::steady_clock::time_point b);
  void dump(const std::string& path, int rank);

 private:
  struct Gpu {
    std::string name;
    int lane;
    cudaEvent_t a, b;
  };
  struct Host {
    std::string name;
    int lane;
    double a_us, b_us;
  };
  cudaEvent_t origin_ = nullptr;
  std::chrono::steady_clock::time_point host_origin_;
  std::mutex mu_;
  std::vector<Gpu> gpu_;
  std::vector<Host> host_;
};

struct Ctx;

/// Host I/O pool -> pinned staging slots -> H2D on the copy stream (the GPU analog of IoPool +
/// DeviceModel::read + decode, scan.cpp:22-93/140-271). Batches are read in order by `threads`
/// workers into a ring of pinned slots; the control thread issues cudaMemcpyAsync per batch and
/// a host callback returns the slot once the copy retires.
class Ingest {
 public:
  Ingest(Ctx& ctx, const std::vector<std::string>& files, const std::vector<BatchPlan>& batches, int threads,
         uint64_t slot_bytes, int nslots);
  ~Ingest();
  /// Blocks until batch i is in pinned memory, writes `extra` bytes (segment descriptors) after
  /// the payload, then enqueues the H2D copy of payload+extra to dst. Returns after enqueueing.
  void copy_to_device(size_t i, void* dst, const void* extra, size_t extra_bytes, cudaStream_t copy_stream);
  /// Whether batch i is already in pinned memory (copy_to_device would not block).
  bool ready(size_t i);
  uint64_t bytes_read() const { return bytes_read_; }
  double wait_s() const { return wait_s_; }

 private:
  struct Slot {
    void* host = nullptr;
    int batch = -1;
    bool ready = false;
  };
  void worker();
  static void CUDART_CB on_copied(void* arg);

  Ctx& ctx_;
  std::vector<std::string> files_;
  std::vector<int> fds_;
  std::vector<std::shared_ptr<const FileMapping>> maps_;  // per file: mapped (memcpy) or null (pread)
  const std::vector<BatchPlan>& batches_;
  uint64_t slot_bytes_;
  std::vector<Slot> slots_;
  std::mutex mu_;
  std::condition_variable cv_;
  size_t next_job_ = 0;
  long cur_batch_ = -1;        // batch whose pieces are being handed out
  size_t cur_ext_ = 0;         // its next extent
  std::vector<int> pending_;   // per batch: pieces being read
  std::vector<int> slot_of_batch_;
  std::deque<int> free_slots_;
  bool stop_ = false;
  std::string error_;
  uint64_t bytes_read_ = 0;
  double wait_s_ = 0;
  std::vector<std::thread> threads_;
  struct CopyDone {
    Ingest* self;
    int slot;
  };
  std::vector<std::unique_ptr<CopyDone>> done_args_;
  cudaStream_t cb_stream_ = nullptr;     // slot-release host callbacks (off the copy stream)
  std::vector<cudaEvent_t> slot_ev_;     // per pinned slot: its copy's completion
};

struct Ctx {
  int device = 0, rank = 0, nranks = 1;
  cudaStream_t compute = nullptr, copy = nullptr, comm = nullptr;
  ncclComm_t nccl = nullptr;
  DevicePool pool;
  FooterCache footers;
  FileMapCache maps;
  int io_threads = 0;
  uint64_t batch_bytes = 64ull << 20;
  int pinned_slots = 0;
  bool semijoin = true;
  // Pinned staging ring (reused across queries).
  std::vector<void*> pinned;
  uint64_t pinned_slot_bytes = 0;
  // Device event-time accounting of the dominant probe kernel.
  cudaEvent_t ev_a = nullptr, ev_b = nullptr;
  // Symmetric heap for the fused NVLink path (nranks > 1): one cudaMalloc'ed region per rank,
  // mapped into every peer with CUDA IPC; per-query bump allocation in identical order on all
  // ranks gives identical offsets, so a peer's table is symm_peer[p] + offset.
  uint8_t* symm = nullptr;
  size_t symm_bytes = 0, symm_top = 0;
  std::vector<uint8_t*> symm_peer;
  bool p2p = false;  // opt-in (psg_ctx_set_fused_shuffle); the NCCL path measured faster for Q3
  bool symm_failed = false;  // CUDA IPC unavailable on some rank (decided collectively)
  void init_symmetric_heap(size_t bytes);  // collective over the NCCL communicator
  void free_symmetric_heap();              // collective (before a re-init)
  void free_symmetric_heap_local();
  // the heap's last kSymmReserve bytes: the peer-barrier flags (one u32 per source rank)
  static constexpr size_t kSymmReserve = 256;
  uint32_t barrier_epoch = 0;  // last peer-barrier epoch (reset with the heap)
  uint32_t* barrier_flags(int peer) const {
    return reinterpret_cast<uint32_t*>(symm_peer[peer] + symm_bytes - kSymmReserve);
  }
  uint8_t* symm_alloc(size_t bytes) {       // nullptr when the heap is exhausted
    const size_t off = (symm_top + 255) & ~size_t(255);
    if (!symm || off + bytes + kSymmReserve > symm_bytes) return nullptr;
    symm_top = off + bytes;
    return symm + off;
  }
  void ensure_pinned(int nslots, uint64_t slot_bytes);
  // mapped pinned words for gathered scalar host reads (launch_gather_words)
  unsigned long long* host_words = nullptr;
  unsigned long long* ensure_host_words();
  Timeline* timeline = nullptr;  // set for the duration of a query when PSG_TIMELINE is on
  bool no_buckets = false;       // set while a query re-runs after a bucket-overflow-list overflow
  bool no_keybits = false;       // set while a query re-runs after a key-bitmap build did not apply
  ~Ctx();
};

/// Process-wide cache of pinned host blocks for result rows: D2H at full PCIe speed without
/// re-pinning (cudaHostAlloc of ~400 MB costs more than the copy) and without zero-filling.
class PinnedBlock {
 public:
  static std::shared_ptr<PinnedBlock> get(size_t bytes);
  ~PinnedBlock();
  void* data() const { return p_; }
  size_t bytes() const { return n_; }

 private:
  void* p_ = nullptr;
  size_t n_ = 0;
};

struct ResultRows {
  Schema schema;
  std::vector<uint64_t> words;          // row-major (small results)
  std::shared_ptr<PinnedBlock> pinned;  // row-major (large results), takes precedence
  uint64_t nrows = 0;
  psg_stats stats{};
  uint64_t* mutable_rows(uint64_t nwords) {
    if (nwords * 8 >= (1u << 20)) {
      pinned = PinnedBlock::get(nwords * 8);
      return static_cast<uint64_t*>(pinned->data());
    }
    words.resize(nwords);
    return words.data();
  }
  const uint64_t* data() const { return pinned ? static_cast<const uint64_t*>(pinned->data()) : words.data(); }
};

struct Staged;  // HBM-resident file images (psg_stage_plan)

ResultRows execute_plan(Ctx& ctx, const std::string& plan_json, const std::string& data_root, int mode,
                        Staged* staged, bool want_rows);
Staged* stage_plan(Ctx& ctx, const std::string& plan_json, const std::string& data_root);
/// Local plans (scan -> replicated joins -> global aggregate, no shuffle; the Q6 analog).
ResultRows execute_local(Ctx& ctx, const std::string& plan_json, const std::string& data_root, int mode);
void free_staged(Staged* s);
/// The plan's storage -> pinned -> HBM pipeline alone (no kernels except block-codec inflate).
ResultRows ingest_only(Ctx& ctx, const std::string& plan_json, const std::string& data_root);

// op adapters (ops.cpp)
struct HostBatch {
  Schema schema;
  std::vector<std::vector<uint64_t>> cols;
  uint64_t rows() const { return cols.empty() ? 0 : cols[0].size(); }
};
HostBatch op_filter(Ctx& ctx, const HostBatch& in, const Predicate& pred);
HostBatch op_partition(Ctx& ctx, const HostBatch& in, const std::string& key, uint32_t nparts, int identity,
                       std::vector<uint64_t>& part_rows);
void op_codec_decompress(Ctx& ctx, int codec, uint64_t n, const void* const* src, const uint64_t* src_len,
                         void* const* dst, const uint64_t* dst_len);
struct GpuHashTable;
GpuHashTable* op_hashtable_build(Ctx& ctx, const std::vector<HostBatch>& batches, const std::string& key_column);
void op_hashtable_free(GpuHashTable* t);
std::vector<uint64_t> op_hashtable_lookup(Ctx& ctx, const GpuHashTable& t, const std::vector<int64_t>& keys,
                                          std::vector<uint64_t>& offsets);
HostBatch op_hashtable_probe(Ctx& ctx, const GpuHashTable& t, const HostBatch& probe, const std::string& probe_key);
const HostBatch& op_hashtable_host(const GpuHashTable& t);  // materialised build side (key_at / payload_at)
HostBatch op_concat(Ctx& ctx, const std::vector<HostBatch>& batches);
HostBatch op_hash_join(Ctx& ctx, const HostBatch& build, const std::string& build_key, const HostBatch& probe,
                       const std::string& probe_key);

// ------------------------------------------------------------ distributed-join microbenchmark
/// JoinVariant (join.hpp:31): blocking, blocking-opt, chunking, deferred.
constexpr int kJoinBlocking = 0, kJoinBlockingOpt = 1, kJoinChunking = 2, kJoinDeferred = 3;
/// One schedule step (PlanStep, join.hpp:70-87): phase, stream (== stream count: the dedicated
/// build stream), wave (-1: none).
struct JoinStep {
  enum class Phase { ConcatLeft, PartitionLeft, SizesLeft, ShuffleLeft, Build, ConcatRight, PartitionRight, SizesRight,
                     ShuffleRight, Probe, Drain };
  Phase phase;
  int stream;
  int wave;
};
std::vector<JoinStep> join_schedule(int variant, int streams, int left_waves, int right_waves);
struct JoinSpecC {
  int variant = kJoinDeferred;
  int stream_count = 2;
  uint64_t chunk_rows = 32 * 1024;
};
/// Host columns of one node's input (key column first).
struct HostTable {
  std::vector<std::string> names;
  std::vector<std::vector<uint64_t>> cols;
  uint64_t rows() const { return cols.empty() ? 0 : cols[0].size(); }
};
struct JoinOutcome {
  double runtime_s = 0, device_ms = 0;
  uint64_t result_rows = 0, bytes_received = 0, left_waves = 0, right_waves = 0, host_syncs = 0;
  std::vector<std::vector<uint64_t>> cols;  // collected result columns (build payload ++ probe)
};
JoinOutcome run_join(Ctx& ctx, const JoinSpecC& spec, const HostTable& build, const HostTable& probe, bool collect);
/// gen_build_table / gen_probe_table (workload.cpp:41-71) of the synthetic join workload, this
/// node's slice (slice_for_node, workload.cpp:73-87).
void synthetic_join_tables(uint64_t seed, uint64_t build_rows, uint64_t probe_rows, int payload_cols, double hit_ratio,
                           int node, int nodes, HostTable& build, HostTable& probe);

void gen_synthetic(const std::string& out_dir, int nodes, int devices, uint64_t seed, Codec codec, uint64_t rg_bytes,
                   uint64_t build_rows, uint64_t probe_rows, int payload_cols, double hit_ratio);
void gen_tpch(const std::string& out_dir, double scale, int nodes, int devices, uint64_t seed, Codec codec,
              uint64_t rg_bytes, int threads);

}  // namespace psg
