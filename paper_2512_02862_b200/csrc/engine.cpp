// execute_plan on B200: the GPU re-design of PlanExecution (/root/reference/proj/src/pipeline.cpp:317-920).
//
// Per rank (one GPU, one host control thread):
//   1. replicated scans -> fused filter/compaction kernel -> CSR hash table per local join
//      (load_replicated, pipeline.cpp:386-428)
//   2. shuffle build side: chunks stream storage -> pinned -> HBM; one fused kernel per chunk batch
//      does predicate + local-join chain + compaction of only the needed columns
//      (scan_chunks + apply_chain, scan.cpp:165-271, pipeline.cpp:431-448); for nranks > 1 each
//      batch is hash-partitioned and exchanged over NCCL (run_waves, pipeline.cpp:662-785); the
//      aggregation table is built from the landed rows (shuffle_build_phase :787-809)
//   3. shuffle probe side: for nranks == 1 one fused kernel per batch does predicate + chain +
//      probe + group-by accumulation in the table slot (shuffle_probe_phase + deliver +
//      HashAggregator::add, :811-837, :874-890, :275-294); for nranks > 1 batches are compacted,
//      (optionally Bloom semi-join filtered), exchanged, then probed on the owner
//   4. finalize: compact groups with hits > 0, radix sort by signed key, emit rows (:892-897).
// Copies run on a copy stream, kernels on the compute stream, NCCL on the comm stream; the host
// waits only where a size is data-dependent (the per-wave count exchange).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <functional>
#include <initializer_list>
#include <numeric>
#include <cstdio>
#include <climits>
#include <cstdlib>
#include <deque>
#include <set>

#include "engine.hpp"
#include "jit.hpp"
#include "shuffle_plan.hpp"

#define PSG_NCCL(call)                                                                              \
  do {                                                                                              \
    ncclResult_t r_ = (call);                                                                       \
    if (r_ != ncclSuccess) throw ::psg::Error(PSG_ERR_NCCL, std::string("nccl: ") + ncclGetErrorString(r_)); \
  } while (0)

namespace psg {

/// The bucketed aggregation's overflow list filled up (extreme key skew): the query is re-run with
/// the table's direct atomic updates (execute_plan), so results never depend on bucket sizing.
struct BucketOverflow : Error {
  BucketOverflow() : Error(PSG_ERR_INTERNAL, "aggregation bucket overflow") {}
};
/// The key-bitmap build found what a rank-indexed table cannot hold (duplicate build keys, keys
/// outside the zone-map range, no keys at all): the query is re-run on the materialising build path.
/// Outbox slack of the peer-slab shuffle: one partly filled 256-word chunk per (warp, destination)
/// of the probe kernel (148 SMs x 64 warps).
constexpr uint64_t kSlabChunkSlack = 148ull * 64 * 256;
struct KeybitsRetry : Error {
  KeybitsRetry() : Error(PSG_ERR_INTERNAL, "key-bitmap build not applicable") {}
};

namespace {

using Clock = std::chrono::steady_clock;
int trace_level() {
  static const int lvl = [] {
    const char* e = std::getenv("PSG_TRACE");
    return e ? std::atoi(e) : 0;
  }();
  return lvl;
}
bool trace_on() { return trace_level() > 0; }
/// A one-GPU aggregation table larger than this gets a membership screen (Bloom filter, or the
/// exact key bitmap / rank-indexed table). PSG_SCREEN_MIN_MB overrides the 48 MB default (0:
/// always - lets small parity cases exercise the bitmap and rank-table paths).
uint64_t screen_min_bytes() {
  static const uint64_t v = [] {
    const char* e = std::getenv("PSG_SCREEN_MIN_MB");
    return (e ? std::strtoull(e, nullptr, 10) : 48ull) << 20;
  }();
  return v;
}
/// PSG_KBITS: 1 (default) = exact key bitmaps at every N, 2 = at N > 1 also when the rank table
/// is off (hashed table + exact screen), 0 = Bloom filters only.
int kbits_mode() {
  static const int v = [] {
    const char* e = std::getenv("PSG_KBITS");
    return e ? std::atoi(e) : 1;
  }();
  return v;
}
/// PSG_RANK_TABLE=0: the hashed aggregation table instead of the rank-indexed one.
bool rank_table_env() {
  static const bool v = [] {
    const char* e = std::getenv("PSG_RANK_TABLE");
    return !(e && e[0] == '0');
  }();
  return v;
}
/// PSG_KEYBITS=0: the build side of a rank-indexed table is materialised and shuffled instead of
/// being scanned straight into the key bitmap.
bool keybits_env() {
  static const bool v = [] {
    const char* e = std::getenv("PSG_KEYBITS");
    return !(e && e[0] == '0');
  }();
  return v;
}
/// PSG_SLAB=0: the NCCL shuffle of packed probe rows instead of the peer-slab stores.
bool slab_env() {
  static const bool v = [] {
    const char* e = std::getenv("PSG_SLAB");
    return !(e && e[0] == '0');
  }();
  return v;
}
#define PSG_TRACE_MSG(...)                  \
  do {                                      \
    if (trace_on()) {                       \
      std::fprintf(stderr, "[psg] " __VA_ARGS__); \
      std::fputc('\n', stderr);             \
    }                                       \
  } while (0)
/// PSG_TRACE=1: phase times with a stream sync at every mark; 2: host timestamps only; 3: CUDA
/// events on the stream + host timestamps, no syncs, printed when the query ends (device time per
/// phase including its idle gaps, next to the host time - where the GPU waits for the host).
struct PhaseTimer {
  Clock::time_point t0 = Clock::now(), last = t0;
  struct Mark {
    const char* what;
    cudaEvent_t ev;
    double host_ms;
  };
  std::vector<Mark> marks;
  cudaStream_t stream0 = nullptr;
  void mark(const char* what, cudaStream_t s) {
    if (!trace_on()) return;
    if (trace_level() == 3) {
      Mark m{what, nullptr, std::chrono::duration<double, std::milli>(Clock::now() - t0).count()};
      cudaEventCreate(&m.ev);
      cudaEventRecord(m.ev, s);
      if (marks.empty()) stream0 = s;
      marks.push_back(m);
      return;
    }
    if (trace_level() == 1) cudaStreamSynchronize(s);  // level 2: host timestamps only
    const auto now = Clock::now();
    std::fprintf(stderr, "[psg] %-28s %8.3f ms (total %8.3f)\n", what,
                 std::chrono::duration<double, std::milli>(now - last).count(),
                 std::chrono::duration<double, std::milli>(now - t0).count());
    last = now;
  }
  ~PhaseTimer() {
    if (marks.empty()) return;
    cudaEventSynchronize(marks.back().ev);
    for (size_t i = 1; i < marks.size(); ++i) {
      float ms = 0;
      cudaEventElapsedTime(&ms, marks[i - 1].ev, marks[i].ev);
      std::fprintf(stderr, "[psg] %-34s device %8.3f ms   host %8.3f ms (at %8.3f)\n", marks[i].what, ms,
                   marks[i].host_ms - marks[i - 1].host_ms, marks[i].host_ms);
    }
    for (auto& m : marks) cudaEventDestroy(m.ev);
    cudaGetLastError();
  }
};
double secs_since(Clock::time_point t0) { return std::chrono::duration<double>(Clock::now() - t0).count(); }

uint64_t pow2_at_least(uint64_t x) {
  uint64_t p = 1;
  while (p < x) p <<= 1;
  return p;
}
int shift_of(uint64_t pow2) {
  int l = 0;
  while ((1ULL << l) < pow2) ++l;
  return 64 - l;
}
uint64_t dbl_bits(double d) {
  uint64_t u;
  std::memcpy(&u, &d, 8);
  return u;
}

// ------------------------------------------------------------------------- plan compilation
struct ColRef {
  int join;  // -1: base projected column; else payload p of chain[join]
  int idx;
  bool operator<(const ColRef& o) const { return join != o.join ? join < o.join : idx < o.idx; }
  bool operator==(const ColRef& o) const { return join == o.join && idx == o.idx; }
};

struct Projected {
  Schema schema;
  std::vector<int> file_idx;
};

/// project (scan.cpp:121-137)
Projected project(const Schema& file, const std::vector<std::string>& columns) {
  Projected p;
  for (size_t c = 0; c < file.size(); ++c)
    if (columns.empty() || std::find(columns.begin(), columns.end(), file.fields[c].name) != columns.end()) {
      p.schema.fields.push_back(file.fields[c]);
      p.file_idx.push_back(static_cast<int>(c));
    }
  for (auto& n : columns)
    if (!p.schema.index_of(n)) throw UnknownColumn(n);
  return p;
}

struct LocalJoinDef {
  const JoinNode* node = nullptr;
  const ScanNode* scan = nullptr;
  Projected proj;
  int key_idx = 0;
  std::vector<int> payload_idx;  // proj indices of payload columns (all non-key), order = p
  int probe_key_stage = 0;       // wire index (before this join) of the probe key
  std::vector<int> needed_payload;  // subset of p needed downstream (filled by analysis)
};

struct SourceDef {
  const ScanNode* scan = nullptr;
  Projected proj;
  std::vector<LocalJoinDef> chain;
  std::vector<std::vector<ColRef>> stage_refs;  // [k] wire refs before join k; [chain.size()] final
  Schema wire;
};

SourceDef make_source(const QueryPlan& plan, FooterCache& fc, const std::string& name) {
  for (const auto& s : plan.scans)
    if (s.table == name) {
      SourceDef d;
      d.scan = &s;
      auto meta = fc.get(s.paths.at(0));
      d.proj = project(meta->schema, s.columns);
      d.wire = d.proj.schema;
      std::vector<ColRef> refs;
      for (size_t i = 0; i < d.wire.size(); ++i) refs.push_back({-1, static_cast<int>(i)});
      d.stage_refs.push_back(refs);
      return d;
    }
  for (const auto& j : plan.joins)
    if (j.id == name) {
      if (j.shuffle) throw InvalidInput("a shuffle join cannot feed another join");
      SourceDef d = make_source(plan, fc, j.probe);
      LocalJoinDef lj;
      lj.node = &j;
      lj.scan = &plan.scan(j.build);
      auto bmeta = fc.get(lj.scan->paths.at(0));
      lj.proj = project(bmeta->schema, lj.scan->columns);
      lj.key_idx = static_cast<int>(lj.proj.schema.require(j.build_key));
      if (lj.proj.schema.fields[lj.key_idx].type != LType::Int64) throw InvalidInput("join key must be int64: " + j.build_key);
      lj.probe_key_stage = static_cast<int>(d.wire.require(j.probe_key));
      if (d.wire.fields[lj.probe_key_stage].type != LType::Int64) throw InvalidInput("probe key must be int64: " + j.probe_key);
      const int jn = static_cast<int>(d.chain.size());
      Schema joined;
      std::vector<ColRef> refs;
      for (size_t c = 0; c < lj.proj.schema.size(); ++c) {
        if (static_cast<int>(c) == lj.key_idx) continue;
        refs.push_back({jn, static_cast<int>(lj.payload_idx.size())});
        lj.payload_idx.push_back(static_cast<int>(c));
        joined.fields.push_back(lj.proj.schema.fields[c]);
      }
      const auto& prev = d.stage_refs.back();
      for (size_t i = 0; i < d.wire.size(); ++i) {
        Field g = d.wire.fields[i];
        if (joined.index_of(g.name)) g.name += "_p";
        joined.fields.push_back(g);
        refs.push_back(prev[i]);
      }
      d.wire = joined;
      d.stage_refs.push_back(refs);
      d.chain.push_back(std::move(lj));
      return d;
    }
  throw InvalidInput("plan references unknown stream: " + name);
}

/// Register map of one fused-kernel program over a source.
struct RegMap {
  std::vector<int> base_proj;  // reg c < n_in -> projected column index
  std::map<ColRef, int> reg_of;
  int n_pred = 0, n_early = 0, n_in = 0, n_regs = 0;
  std::vector<std::vector<int>> payload_regs;  // [join][k] reg of needed payload k
  std::vector<std::vector<int>> payload_cols;  // [join][k] payload p
};

/// Decides which columns a program loads, in which phase. `needed` are final-wire columns the
/// sink consumes; `early_wire` (sink key) must be loaded before the sink's probe.
RegMap analyse(SourceDef& s, const std::vector<int>& needed, int early_wire, bool with_joins) {
  RegMap m;
  const auto& fin = s.stage_refs.back();
  std::set<ColRef> need;
  for (int w : needed) need.insert(fin[w]);
  std::set<ColRef> early;
  if (early_wire >= 0) early.insert(fin[early_wire]);
  if (with_joins)
    for (size_t j = 0; j < s.chain.size(); ++j) {
      const ColRef k = s.stage_refs[j][s.chain[j].probe_key_stage];
      need.insert(k);
      early.insert(k);
    }
  // predicate columns first
  for (const auto& a : s.scan->predicate) {
    const int pi = static_cast<int>(s.proj.schema.require(a.column));
    if (!m.reg_of.count({-1, pi})) {
      m.reg_of[{-1, pi}] = static_cast<int>(m.base_proj.size());
      m.base_proj.push_back(pi);
    }
  }
  m.n_pred = static_cast<int>(m.base_proj.size());
  for (const auto& r : early)
    if (r.join < 0 && !m.reg_of.count(r)) {
      m.reg_of[r] = static_cast<int>(m.base_proj.size());
      m.base_proj.push_back(r.idx);
    }
  m.n_early = static_cast<int>(m.base_proj.size());
  for (const auto& r : need)
    if (r.join < 0 && !m.reg_of.count(r)) {
      m.reg_of[r] = static_cast<int>(m.base_proj.size());
      m.base_proj.push_back(r.idx);
    }
  m.n_in = static_cast<int>(m.base_proj.size());
  int reg = m.n_in;
  m.payload_regs.resize(s.chain.size());
  m.payload_cols.resize(s.chain.size());
  for (size_t j = 0; j < s.chain.size(); ++j) {
    for (const auto& r : need)
      if (r.join == static_cast<int>(j)) {
        m.reg_of[r] = reg;
        m.payload_regs[j].push_back(reg++);
        m.payload_cols[j].push_back(r.idx);
      }
  }
  m.n_regs = reg;
  if (m.n_in > kMaxIn || m.n_regs > kMaxRegs) throw InvalidInput("plan touches too many columns for one fused program");
  return m;
}

// ------------------------------------------------------------------------ batch planning
struct ScanBatches {
  std::vector<BatchPlan> batches;
  uint64_t total_rows = 0;
  uint64_t total_bytes = 0;    // H2D footprint
  uint64_t total_dbytes = 0;   // decoded footprint (block codec)
  uint64_t total_payload = 0;  // file bytes
  uint64_t total_scan = 0;     // bytes the scan kernel reads
  uint64_t max_batch_bytes = 0, max_dbytes = 0;
  uint64_t max_segs = 0, max_jobs = 0;
  bool inflate = false;
};

/// Groups surviving row groups of each file into batches of <= batch_bytes packed column chunks.
/// Block-codec files keep their chunks compressed on the wire (the GPU inflates them in HBM,
/// replacing codec_decompress in decode_group, scan.cpp:139-160); such a batch is also capped at
/// 4 x batch_bytes of decoded columns.
ScanBatches plan_batches(FooterCache& fc, const ScanNode& scan, const std::vector<int>& file_cols, int file_base,
                         uint64_t batch_bytes) {
  ScanBatches out;
  for (size_t f = 0; f < scan.paths.size(); ++f) {
    auto meta = fc.get(scan.paths[f]);
    const bool block = meta->codec == Codec::Block;
    const auto groups = prune(*meta, scan.predicate);
    BatchPlan cur;
    cur.file = file_base + static_cast<int>(f);
    cur.inflate = block;
    auto flush = [&] {
      if (cur.groups.empty()) return;
      cur.bytes += 16;  // tail padding: 16-byte async copies may read 8 bytes past the last chunk
      if (block) {
        cur.dbytes += 16;
        // longest streams first: the decoders of one warp finish together
        std::sort(cur.jobs.begin(), cur.jobs.end(), [](const BatchPlan::Job& a, const BatchPlan::Job& b) {
          return a.csize != b.csize ? a.csize > b.csize : a.src_off < b.src_off;
        });
      }
      out.total_rows += cur.total_rows;
      out.total_bytes += cur.bytes;
      out.total_dbytes += cur.dbytes;
      out.total_payload += cur.payload_bytes;
      out.total_scan += cur.scan_bytes();
      out.max_batch_bytes = std::max(out.max_batch_bytes, cur.bytes);
      out.max_dbytes = std::max(out.max_dbytes, cur.dbytes);
      out.max_segs = std::max<uint64_t>(out.max_segs, cur.groups.size());
      out.max_jobs = std::max<uint64_t>(out.max_jobs, cur.jobs.size());
      out.inflate = out.inflate || block;
      out.batches.push_back(std::move(cur));
      cur = BatchPlan{};
      cur.file = file_base + static_cast<int>(f);
      cur.inflate = block;
    };
    for (size_t g : groups) {
      const GroupMeta& gm = meta->groups[g];
      uint64_t gbytes = 0, gdbytes = 0;
      for (int c : file_cols) gbytes += gm.cols[c].csize, gdbytes += gm.cols[c].usize;
      if (!cur.groups.empty() &&
          (cur.bytes + gbytes > batch_bytes || (block && cur.dbytes + gdbytes > 4 * batch_bytes)))
        flush();
      // chunks of this group in file order, packed; merge adjacent extents
      std::vector<std::pair<uint64_t, int>> order;
      for (size_t k = 0; k < file_cols.size(); ++k) order.push_back({gm.cols[file_cols[k]].offset, static_cast<int>(k)});
      std::sort(order.begin(), order.end());
      std::vector<uint64_t> pos(file_cols.size());
      for (auto& [off, k] : order) {
        const ChunkMeta& ch = gm.cols[file_cols[k]];
        const uint64_t len = ch.csize;
        // 16-byte aligned chunk positions (vector loads in the fused kernel, aligned words in the
        // inflate bit reader); padding breaks an extent
        cur.bytes = (cur.bytes + 15) & ~15ULL;
        if (block) {
          if (ch.csize > 0xFFFFFFFFull || ch.usize > 0xFFFFFFFFull)
            throw InvalidInput("block-codec column chunk larger than 4 GiB: " + scan.paths[f]);
          cur.dbytes = (cur.dbytes + 15) & ~15ULL;
          cur.jobs.push_back({cur.bytes, cur.dbytes, static_cast<uint32_t>(ch.csize), static_cast<uint32_t>(ch.usize)});
          pos[k] = cur.dbytes;
          cur.dbytes += ch.usize;
          cur.ubytes += ch.usize;
        } else {
          pos[k] = cur.bytes;
        }
        cur.payload_bytes += len;
        if (!cur.extents.empty() && cur.extents.back().file_off + cur.extents.back().len == off &&
            cur.extents.back().buf_off + cur.extents.back().len == cur.bytes)
          cur.extents.back().len += len;
        else
          cur.extents.push_back({off, len, cur.bytes});
        cur.bytes += len;
      }
      cur.groups.push_back(g);
      cur.rows.push_back(gm.rows);
      cur.bytes = (cur.bytes + 15) & ~15ULL;
      cur.pos.push_back(std::move(pos));
      cur.total_rows += gm.rows;
    }
    flush();
  }
  return out;
}

/// Device inflate jobs of a block-codec batch whose compressed image is at `cbase` and whose
/// decoded image goes to `dbase`.
std::vector<InflateJob> inflate_jobs(const BatchPlan& b, uint8_t* cbase, uint8_t* dbase) {
  std::vector<InflateJob> jobs(b.jobs.size());
  for (size_t i = 0; i < b.jobs.size(); ++i)
    jobs[i] = InflateJob{cbase + b.jobs[i].src_off, dbase + b.jobs[i].dst_off, b.jobs[i].csize, b.jobs[i].usize};
  return jobs;
}

/// Segment descriptors of a batch placed at device address `dev_base`.
std::vector<Segment> make_segments(const BatchPlan& b, uint8_t* dev_base, uint64_t& tiles) {
  std::vector<Segment> segs(b.groups.size());
  const uint64_t T = static_cast<uint64_t>(scan_tile_rows());
  tiles = 0;
  for (size_t i = 0; i < b.groups.size(); ++i) {
    Segment& s = segs[i];
    std::memset(&s, 0, sizeof s);
    for (size_t k = 0; k < b.pos[i].size(); ++k) s.col[k] = reinterpret_cast<const uint64_t*>(dev_base + b.pos[i][k]);
    s.rows = b.rows[i];
    s.tile_begin = tiles;
    tiles += (b.rows[i] + T - 1) / T;
  }
  return segs;
}

/// tile -> segment index table for k_scan (segments must have tile_begin set).
std::vector<uint32_t> tile_table(const std::vector<Segment>& segs) {
  const uint64_t T = static_cast<uint64_t>(scan_tile_rows());
  std::vector<uint32_t> t;
  for (size_t i = 0; i < segs.size(); ++i) {
    const uint64_t n = (segs[i].rows + T - 1) / T;
    t.insert(t.end(), n, static_cast<uint32_t>(i));
  }
  return t;
}

/// Segment array followed by its tile table, as one host blob (8-byte aligned).
std::vector<uint8_t> pack_view(const std::vector<Segment>& segs, size_t& tile_off) {
  auto tt = tile_table(segs);
  tile_off = segs.size() * sizeof(Segment);
  std::vector<uint8_t> blob(tile_off + ((tt.size() * 4 + 7) & ~size_t(7)));
  std::memcpy(blob.data(), segs.data(), tile_off);
  std::memcpy(blob.data() + tile_off, tt.data(), tt.size() * 4);
  return blob;
}

// --------------------------------------------------------------------------- device views
struct BatchView {
  const Segment* d_segs = nullptr;
  const uint32_t* d_tile_seg = nullptr;
  int nsegs = 0;
  uint64_t ntiles = 0;
  uint64_t rows = 0;   // upper bound (input rows)
  uint64_t bytes = 0;  // algorithmic input bytes (column chunks scanned)
};

/// Materialised columnar batch in HBM (needed columns only).
struct DevCols {
  std::vector<DevBuf> cols;
  DevBuf count;  // unsigned long long row counter
  uint64_t cap = 0;
  uint64_t rows = 0;  // host copy once known
};

}  // namespace

// ------------------------------------------------------------------------------ Staged
struct StagedScan {
  uint64_t payload = 0;
  DevBuf data;
  DevBuf segs;  // segment array + tile table at tile_off
  size_t tile_off = 0;
  int nsegs = 0;
  uint64_t ntiles = 0, rows = 0, bytes = 0;
  std::vector<Segment> host_segs;  // the same segments on the host (chunked probe pipeline)
};
struct Staged {
  std::string plan_json, data_root;
  std::map<std::string, StagedScan> scans;  // key: "table|cols"
  uint64_t bytes = 0;  // decoded column-chunk bytes the scans read
  uint64_t h2d = 0;    // bytes copied host->HBM while staging
};

namespace {

std::string scan_key(const ScanNode& s, const std::vector<int>& file_cols) {
  std::string k = s.table + "|";
  for (int c : file_cols) k += std::to_string(c) + ",";
  return k;
}

// ------------------------------------------------------------------------ the executor
struct StreamSession;
class Execution {
 public:
  struct Feed;
  Execution(Ctx& ctx, const std::string& plan_json, const std::string& data_root, int mode, Staged* staged)
      : ctx_(ctx), mode_(mode), staged_(staged), plan_(QueryPlan::from_json_text(plan_json, data_root, ctx.rank, ctx.nranks)) {}
  ~Execution() {
    if (build_pending_) cudaStreamSynchronize(ctx_.comm);  // (error paths) before the tables go
    for (auto& e : timed_) cudaEventDestroy(e.first), cudaEventDestroy(e.second);
  }

  ResultRows run(bool want_rows);
  // local plans (no shuffle): scan -> replicated joins -> global aggregate (the Q6 analog)
  ResultRows run_local();
  // staging entry: read every scan's needed chunks into HBM
  void stage(Staged& st);
  // storage -> pinned -> HBM of every chunk the plan reads, through the same ingest session as
  // run(), with no kernels (block codec: + inflate): the ingest term of the e2e roofline
  ResultRows run_ingest_only();

 private:
  // ---- compilation ----
  void compile();
  std::vector<int> file_cols_of(const SourceDef& s, const RegMap& m) const {
    std::vector<int> fc;
    for (int p : m.base_proj) fc.push_back(s.proj.file_idx[p]);
    return fc;
  }

  // ---- feeds ----
  std::unique_ptr<Feed> open_feed(const ScanNode& scan, const std::vector<int>& file_cols);

  // ---- stages ----
  void build_local_tables();
  ScanProgram base_program(const SourceDef& s, const RegMap& m, bool with_joins);
  // aligned: v is a feed batch (16-byte aligned PSTO chunks with tail padding; bulk copies allowed)
  void materialize_into(DevCols& out, const ScanProgram& p0, const BatchView& v, const std::vector<int>& out_regs,
                        int part_key_reg, DevBuf* part_counts, bool timed = false, bool aligned = false);
  DevCols alloc_cols(size_t ncols, uint64_t cap);
  // Local joins whose build side repeats keys (HashTable::build keeps duplicates and probe emits
  // every match, ops.cpp:105-222, apply_chain pipeline.cpp:431-448): the chain cannot stay in
  // registers, so the batch is compacted first (predicate only) and each join then expands it
  // (count -> exclusive scan -> write; payload ++ probe columns like ops.cpp:193-200).
  bool dup_chain(const SourceDef& s) const;
  DevCols materialize_chain(const SourceDef& s, const RegMap& m, const BatchView& v, const std::vector<int>& out_regs);
  DevCols concat_cols(std::vector<DevCols>& parts, size_t ncols);
  uint64_t read_count(DevCols& c);
  // duplicate flags of local semi-join bitmaps built optimistically (SINK_KEYBITS), [rows, flag]
  // each: enqueue their reads before a host sync the query makes anyway, then check
  std::vector<DevBuf> lt_flags_;
  std::vector<uint64_t> lt_flag_host_;
  void enqueue_lt_flags() {
    lt_flag_host_.assign(2 * lt_flags_.size(), 0);
    for (size_t i = 0; i < lt_flags_.size(); ++i)
      PSG_CUDA(cudaMemcpyAsync(lt_flag_host_.data() + 2 * i, lt_flags_[i].p, 16, cudaMemcpyDeviceToHost, ctx_.compute));
  }
  void check_lt_flags() {  // after the sync that completed enqueue_lt_flags' copies
    for (size_t i = 0; i < lt_flags_.size(); ++i)
      if (lt_flag_host_[2 * i + 1] != 0) throw KeybitsRetry();
    lt_flags_.clear();
  }
  /// One gathered host read of device scalars (u32 where the flag says so) plus the pending
  /// local-table duplicate flags: one small kernel writing mapped pinned memory and one stream
  /// sync, then the flag check.
  void read_words(std::initializer_list<std::pair<const void*, bool>> srcs, uint64_t* out) {
    GatherWords g{};
    for (const auto& [ptr, is32] : srcs) {
      if (is32) g.w32 |= 1u << g.n;
      g.src[g.n++] = ptr;
    }
    const int nw = g.n;
    if (nw + static_cast<int>(lt_flags_.size()) + 1 > 24) throw Error(PSG_ERR_INTERNAL, "read_words: too many words");
    if (barrier_err_.p) {  // a peer barrier that timed out (a rank never arrived)
      g.w32 |= 1u << g.n;
      g.src[g.n++] = barrier_err_.p;
    }
    const int nb = g.n;
    for (auto& f : lt_flags_) g.src[g.n++] = f.as<unsigned long long>() + 1;
    unsigned long long* hw = ctx_.ensure_host_words();
    launch_gather_words(g, hw, ctx_.compute);
    PSG_CUDA(cudaStreamSynchronize(ctx_.compute));
    const volatile unsigned long long* v = hw;
    for (int i = 0; i < nw; ++i) out[i] = v[i];
    if (nb > nw && v[nw] != 0) throw Error(PSG_ERR_NCCL, "peer barrier timed out (a rank did not arrive)");
    for (int i = nb; i < g.n; ++i)
      if (v[i] != 0) throw KeybitsRetry();
    lt_flags_.clear();
  }
  // event pairs around the timed (dominant) kernel launches, resolved after the query's last sync
  // (no host sync per launch)
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> timed_;
  void resolve_timed() {
    for (auto& e : timed_) {
      float ms = 0;
      PSG_CUDA(cudaEventElapsedTime(&ms, e.first, e.second));
      st_.probe_kernel_ms += ms;
      cudaEventDestroy(e.first), cudaEventDestroy(e.second);
    }
    timed_.clear();
  }
  /// Widens [lo, hi] by the footer zone maps of column fcol over the files (cached per footer).
  void zone_range(const std::vector<std::string>& paths, int fcol, long long& lo, long long& hi) {
    for (const auto& path : paths) {
      auto m = ctx_.footers.get(path);
      if (fcol < 0 || static_cast<size_t>(fcol) >= m->zmin.size()) continue;
      lo = std::min<long long>(lo, m->zmin[fcol]);
      hi = std::max<long long>(hi, m->zmax[fcol]);
    }
  }
  void run_scan(const ScanProgram& p, const BatchView& v, bool timed, cudaStream_t stream = nullptr);

  // shuffle (nranks > 1)
  struct Received {
    DevBuf buf;
    std::vector<Segment> segs;  // host descriptors
    uint64_t rows = 0;
  };
  Received exchange(DevCols& mat, int ncols, int key_col, DevBuf& part_counts, bool have_data,
                    KeyField kf = KeyField{0, 0, 0}, cudaStream_t stream = nullptr);
  BatchView upload_segments(std::vector<Segment> segs, DevBuf& holder, cudaStream_t stream = nullptr);

  void build_agg_table(uint64_t build_rows, uint64_t bloom_words, uint64_t rank_slots = 0);
  void pack_accumulators();
  bool build_symmetric_agg_table(uint64_t max_rows, bool bloom);
  void gpu_barrier();
  void finalize_grouped(ResultRows& out, bool want_rows);
  void finalize_global(ResultRows& out);

  Ctx& ctx_;
  int mode_;
  Staged* staged_;
  QueryPlan plan_;
  const JoinNode* shuffle_ = nullptr;
  SourceDef bsrc_, psrc_;
  bool agg_ = false, grouped_ = false;
  // aggregate column resolution
  std::vector<int> probe_sum_wire, build_sum_wire;  // wire idx per side
  std::vector<std::pair<int, int>> sum_order;       // (side 0 build/1 probe, k) in agg.sums order
  Schema result_schema_;
  // local tables
  struct LocalTable {
    DevBuf keys, cnt, start, bitmap;
    std::vector<DevBuf> payload;
    uint64_t cap = 0;
    bool unique = true;
    LocalTableDev dev{};
  };
  std::vector<std::unique_ptr<LocalTable>> bl_tables_, pl_tables_;
  // agg table
  DevBuf agg_hot_, agg_cold_, agg_bloom_, agg_dups_, agg_kbits_, agg_krank_, agg_krec_, global_acc_, barrier_word_, barrier_err_;
  DevBuf bkt_, bkt_fill_, bkt_ovf_, bkt_ovf_count_;  // bucketed aggregation (rank table, one GPU)
  bool bucket_mode_ = false;
  BucketDev bd_{};
  uint64_t nbuckets_ = 0;
  /// Bucketed aggregation; at N > 1 (peer-slab shuffle) the probe sums' value ranges are the
  /// all-reduced ones (prange_lo/hi, probe_sum_wire order) and probe_rows the global total, so
  /// every rank encodes alike and sizes its buckets for the rows it will own.
  bool setup_buckets(const int64_t* prange_lo = nullptr, const int64_t* prange_hi = nullptr, uint64_t probe_rows_all = 0);
  /// Symmetric heap of at least `bytes` (collective; every rank passes the same value).
  bool ensure_symmetric(size_t bytes);
  // peer-slab shuffle (N > 1): counters and receive slab in the symmetric heap
  bool slab_mode_ = false;
  PackLayout slab_pack_;
  uint64_t slab_cap_ = 0;
  size_t slab_cnt_off_ = 0, slab_off_ = 0;
  DevBuf slab_recv_;
  DevBuf slab_grec_;  // {global bitmap word, own rank} records (ScanProgram::slab_grec)
  void apply_buckets(ScanProgram& p) const;
  void finalize_buckets(ResultRows& out, bool want_rows);
  AggTableDev aggt_{};
  // the build insert running on ctx_.comm concurrently with the probe side (N > 1 Bloom path)
  struct Event {
    cudaEvent_t e = nullptr;
    Event() { cudaEventCreateWithFlags(&e, cudaEventDisableTiming); }
    ~Event() {
      if (e) cudaEventDestroy(e);
    }
    Event(const Event&) = delete;
    Event& operator=(const Event&) = delete;
    cudaEvent_t get() const { return e; }
  };
  Event build_fork_, build_done_;
  bool build_pending_ = false;
  // timed shuffle send/recv groups (psg_stats.exchange_ms, summed once the query has drained)
  struct TimedPair {
    cudaEvent_t a = nullptr, b = nullptr;
    TimedPair() {
      cudaEventCreate(&a);
      cudaEventCreate(&b);
    }
    ~TimedPair() {
      cudaEventDestroy(a);
      cudaEventDestroy(b);
    }
    TimedPair(const TimedPair&) = delete;
    TimedPair& operator=(const TimedPair&) = delete;
  };
  std::vector<std::unique_ptr<TimedPair>> xfer_ev_;
  void sum_exchange_time() {
    double ms = 0;
    for (auto& t : xfer_ev_) {
      float x = 0;
      if (cudaEventElapsedTime(&x, t->a, t->b) == cudaSuccess) ms += x;
    }
    cudaGetLastError();
    st_.exchange_ms = ms;
  }
  uint64_t agg_cap_ = 0;
  // stats
  psg_stats st_{};
  uint64_t launches0_ = 0, jit0_ = 0;
  std::vector<std::string> files_;
  std::map<std::string, int> file_index_;
  std::vector<DevBuf> keep_;  // buffers that must live until the end
  std::vector<std::vector<uint8_t>> host_keep_;  // host sources of in-flight async copies
  std::unique_ptr<StreamSession> session_;
  /// (scan, file columns) of every scan in consumption order: replicated scans of the build
  /// chain, of the probe chain, then the shuffle build and probe sources.
  std::vector<std::pair<const ScanNode*, std::vector<int>>> scan_list(const RegMap& bm, const RegMap& pm);
};

// ------------------------------------------------------------------------------ feeds
struct Execution::Feed {
  virtual ~Feed() = default;
  virtual bool next(BatchView& v) = 0;
  virtual void done() = 0;
  /// Staged scans: the segments on the host (nullptr when streaming).
  virtual const std::vector<Segment>* host_segments() const { return nullptr; }
  uint64_t total_rows = 0;
  size_t nbatches = 0;
};

/// One ingest session per query: every batch of every scan the query streams (in consumption
/// order: replicated scans, shuffle build side, probe side) goes through one I/O pool, one pinned
/// ring and one ring of HBM slots, so reads of the next scan overlap the processing of the
/// current one (the reference's reader combining, scan.cpp:22-93, without phase bubbles).
struct StreamSession {
  Ctx& ctx;
  std::vector<std::string> files;
  std::map<std::string, int> file_index;
  std::vector<BatchPlan> batches;
  struct Range {
    size_t begin = 0, end = 0;
    uint64_t rows = 0;
  };
  std::map<std::string, std::deque<Range>> ranges;  // scan_key -> batch ranges in consumption order
  std::unique_ptr<Ingest> ingest;
  std::vector<DevBuf> slots;
  std::vector<cudaEvent_t> slot_free, copied;
  uint64_t slot_bytes = 0;
  // block codec: decoded images, per-slot inflate streams, session error word
  std::vector<DevBuf> dslots;
  std::vector<cudaStream_t> istreams;
  std::vector<cudaEvent_t> inflated;
  DevBuf inflate_err;
  uint64_t dslot_bytes = 0;
  uint64_t h2d_bytes = 0;
  int regulated_slots = 0;
  size_t cursor = 0;    // next batch to consume (global order)
  size_t enqueued = 0;  // batches whose copy (+ inflate) has been enqueued
  size_t released = 0;  // batches the consumer has released (slot_free recorded)
  std::vector<BatchView> views;  // per ring slot
  int cur_slot = -1;
  int tl_consume = -1;  // timeline interval of the batch being consumed

  /// budget/ht_reserve: plan memory_budget_bytes and the bytes set aside for hash tables; the ring
  /// depth is regulated to fit (regulate, pipeline.cpp:198-240): InfeasibleBudget when not even one
  /// chunk batch fits, like a queue that cannot hold one chunk.
  StreamSession(Ctx& c, const std::vector<std::pair<const ScanNode*, std::vector<int>>>& scans, uint64_t budget = 0,
                uint64_t ht_reserve = 0)
      : ctx(c) {
    uint64_t max_bytes = 0, max_segs = 0, max_dbytes = 0, max_jobs = 0;
    for (auto& [scan, fcols] : scans) {
      const std::string key = scan_key(*scan, fcols);
      // union file list; plan this scan's batches against it
      std::vector<int> idx;
      for (auto& path : scan->paths) {
        auto it = file_index.find(path);
        if (it == file_index.end()) {
          it = file_index.emplace(path, static_cast<int>(files.size())).first;
          files.push_back(path);
        }
        idx.push_back(it->second);
      }
      ScanBatches sb = plan_batches(ctx.footers, *scan, fcols, 0, ctx.batch_bytes);
      Range r;
      r.begin = batches.size();
      for (auto& bp : sb.batches) {
        bp.file = idx[bp.file];
        batches.push_back(std::move(bp));
      }
      r.end = batches.size();
      r.rows = sb.total_rows;
      ranges[key].push_back(r);
      max_bytes = std::max(max_bytes, sb.max_batch_bytes);
      max_segs = std::max(max_segs, sb.max_segs);
      max_dbytes = std::max(max_dbytes, sb.max_dbytes);
      max_jobs = std::max(max_jobs, sb.max_jobs);
    }
    if (batches.empty()) return;
    const uint64_t T = static_cast<uint64_t>(scan_tile_rows());
    const uint64_t cap = std::max(max_bytes, ctx.batch_bytes);
    const uint64_t max_tiles = std::max(cap, max_dbytes) / 8 / T + max_segs + 1;
    slot_bytes = (cap + max_segs * sizeof(Segment) + max_tiles * 4 + max_jobs * sizeof(InflateJob) + 4096 + 4095) &
                 ~4095ULL;
    dslot_bytes = (max_dbytes + 4095) & ~4095ULL;
    const int threads = std::max(1, ctx.io_threads);
    const int pinned = ctx.pinned_slots > 0 ? ctx.pinned_slots : threads * 2 + 2;
    ingest = std::make_unique<Ingest>(ctx, files, batches, threads, slot_bytes, pinned);
    // HBM ring depth: batches in flight between the readers and the scan. PSG_RING_SLOTS
    // overrides it (measurement knob).
    static const int ring_env = [] {
      const char* e = std::getenv("PSG_RING_SLOTS");
      return e ? std::atoi(e) : 0;
    }();
    int nd = static_cast<int>(std::min<size_t>(batches.size(), ring_env > 0 ? ring_env : 8));
    const uint64_t per_slot = slot_bytes + dslot_bytes;
    if (budget) {
      const uint64_t fixed = ht_reserve + 2 * std::max(slot_bytes, dslot_bytes);  // tables + materialisation transients
      if (fixed >= budget)
        throw InfeasibleBudget("fixed residents (" + std::to_string(fixed) + " bytes) leave no room for the chunk ring in a budget of " +
                               std::to_string(budget));
      const uint64_t fit = (budget - fixed) / per_slot;
      if (fit < 1)
        throw InfeasibleBudget("the chunk ring cannot hold even one batch of " + std::to_string(per_slot) + " bytes");
      nd = static_cast<int>(std::min<uint64_t>(static_cast<uint64_t>(nd), fit));
    }
    regulated_slots = nd;
    for (int k = 0; k < nd; ++k) {
      slots.emplace_back(ctx.pool, slot_bytes, ctx.copy);
      cudaEvent_t x, y;
      PSG_CUDA(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
      PSG_CUDA(cudaEventCreateWithFlags(&y, cudaEventDisableTiming));
      slot_free.push_back(x);
      copied.push_back(y);
      if (dslot_bytes) {
        // decoded images + one inflate stream per slot: batches decode concurrently (one thread
        // per chunk, so a single batch fills only part of the GPU)
        dslots.emplace_back(ctx.pool, dslot_bytes, ctx.copy);
        cudaStream_t is;
        PSG_CUDA(cudaStreamCreateWithFlags(&is, cudaStreamNonBlocking));
        istreams.push_back(is);
        PSG_CUDA(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
        inflated.push_back(x);
      }
    }
    views.resize(slots.size());
    if (dslot_bytes) {
      inflate_err = DevBuf(ctx.pool, sizeof(unsigned int), ctx.copy);
      PSG_CUDA(cudaMemsetAsync(inflate_err.p, 0, sizeof(unsigned int), ctx.copy));
    }
  }
  ~StreamSession() {
    cudaStreamSynchronize(ctx.copy);
    for (auto is : istreams) cudaStreamSynchronize(is);
    cudaStreamSynchronize(ctx.compute);
    ingest.reset();
    for (auto x : slot_free) cudaEventDestroy(x);
    for (auto x : copied) cudaEventDestroy(x);
    for (auto x : inflated) cudaEventDestroy(x);
    for (auto is : istreams) cudaStreamDestroy(is);
  }
  /// Raises IoFailure when any chunk of the session failed to inflate (codec_decompress,
  /// psto.cpp:138-140). Call after the compute stream has drained.
  void check_inflate() {
    if (!inflate_err.p) return;
    unsigned int e = 0;
    PSG_CUDA(cudaMemcpy(&e, inflate_err.p, sizeof e, cudaMemcpyDeviceToHost));
    if (e) throw IoFailure("inflate failed");
  }
  /// Enqueues batch j's host->HBM copy (and inflate) into its ring slot. The slot's previous
  /// occupant (batch j - nslots) must have been released (its slot_free event recorded).
  void enqueue(size_t j) {
    const int k = static_cast<int>(j % slots.size());
    const BatchPlan& b = batches[j];
    auto* base = slots[k].as<uint8_t>();
    uint8_t* dbase = b.inflate ? dslots[k].as<uint8_t>() : base;
    uint64_t nt = 0;
    auto segs = make_segments(b, dbase, nt);
    if (j >= slots.size()) PSG_CUDA(cudaStreamWaitEvent(ctx.copy, slot_free[k], 0));
    size_t toff = 0;
    auto blob = pack_view(segs, toff);
    size_t joff = blob.size();
    if (b.inflate) {
      auto jobs = inflate_jobs(b, base, dbase);
      blob.resize(joff + jobs.size() * sizeof(InflateJob));
      std::memcpy(blob.data() + joff, jobs.data(), jobs.size() * sizeof(InflateJob));
    }
    ingest->copy_to_device(j, base, blob.data(), blob.size(), ctx.copy);  // timeline lane 1 inside
    h2d_bytes += b.bytes + blob.size();
    PSG_CUDA(cudaEventRecord(copied[k], ctx.copy));
    if (b.inflate) {
      PSG_CUDA(cudaStreamWaitEvent(istreams[k], copied[k], 0));
      const int ti = ctx.timeline ? ctx.timeline->gpu_begin("inflate b" + std::to_string(j), 2, istreams[k]) : -1;
      launch_inflate(reinterpret_cast<const InflateJob*>(base + b.bytes + joff), static_cast<uint32_t>(b.jobs.size()),
                     inflate_err.as<unsigned int>(), istreams[k]);
      if (ti >= 0) ctx.timeline->gpu_end(ti, istreams[k]);
      PSG_CUDA(cudaEventRecord(inflated[k], istreams[k]));
    }
    BatchView& v = views[k];
    v.d_segs = reinterpret_cast<const Segment*>(base + b.bytes);
    v.d_tile_seg = reinterpret_cast<const uint32_t*>(base + b.bytes + toff);
    v.nsegs = static_cast<int>(segs.size());
    v.ntiles = nt;
    v.rows = b.total_rows;
    v.bytes = b.scan_bytes();
    ++enqueued;
  }
  /// Read-ahead: enqueue the copies (and inflates) of upcoming batches whose bytes are already
  /// in pinned memory and whose ring slot is free, so transfers and decoding run ahead of the
  /// consumer even when it blocks on the host (the per-wave exchange sync at N > 1).
  void read_ahead() {
    while (enqueued < batches.size() && enqueued < released + slots.size() && ingest->ready(enqueued)) enqueue(enqueued);
  }
  /// Stages batch i (must be the next in consumption order) into its HBM ring slot.
  void stage(size_t i, BatchView& v) {
    if (i != cursor) throw Error(PSG_ERR_INTERNAL, "ingest batches consumed out of order");
    while (enqueued <= i) enqueue(enqueued);  // blocks on the read of batch i if needed
    const int k = static_cast<int>(i % slots.size());
    PSG_CUDA(cudaStreamWaitEvent(ctx.compute, batches[i].inflate ? inflated[k] : copied[k], 0));
    if (ctx.timeline) tl_consume = ctx.timeline->gpu_begin("compute b" + std::to_string(i), 3, ctx.compute);
    v = views[k];
    cur_slot = k;
    ++cursor;
    read_ahead();
  }
  void release() {
    if (cur_slot >= 0) {
      if (tl_consume >= 0) ctx.timeline->gpu_end(tl_consume, ctx.compute), tl_consume = -1;
      PSG_CUDA(cudaEventRecord(slot_free[cur_slot], ctx.compute));
      ++released;
      cur_slot = -1;
      read_ahead();
    }
  }
};

struct SessionFeed : Execution::Feed {
  StreamSession& ss;
  size_t i, end;
  SessionFeed(StreamSession& s, const StreamSession::Range& r) : ss(s), i(r.begin), end(r.end) {
    total_rows = r.rows;
    nbatches = r.end - r.begin;
  }
  bool next(BatchView& v) override {
    if (i >= end) return false;
    ss.stage(i++, v);
    return true;
  }
  void done() override { ss.release(); }
};

/// One batch covering a scan's staged HBM image.
struct StagedFeed : Execution::Feed {
  const StagedScan* s;
  bool given = false;
  explicit StagedFeed(const StagedScan* sc) : s(sc) {
    total_rows = sc->rows;
    nbatches = sc->nsegs ? 1 : 0;
  }
  bool next(BatchView& v) override {
    if (given || s->nsegs == 0) return false;
    given = true;
    v.d_segs = s->segs.as<Segment>();
    v.d_tile_seg = reinterpret_cast<const uint32_t*>(s->segs.as<uint8_t>() + s->tile_off);
    v.nsegs = s->nsegs;
    v.ntiles = s->ntiles;
    v.rows = s->rows;
    v.bytes = s->payload;
    return true;
  }
  void done() override {}
  const std::vector<Segment>* host_segments() const override { return &s->host_segs; }
};

std::unique_ptr<Execution::Feed> Execution::open_feed(const ScanNode& scan, const std::vector<int>& file_cols) {
  if (staged_) {
    auto it = staged_->scans.find(scan_key(scan, file_cols));
    if (it == staged_->scans.end()) throw InvalidInput("staged data does not cover scan " + scan.table);
    return std::make_unique<StagedFeed>(&it->second);
  }
  if (!session_) throw Error(PSG_ERR_INTERNAL, "no ingest session");
  auto it = session_->ranges.find(scan_key(scan, file_cols));
  if (it == session_->ranges.end() || it->second.empty())
    throw Error(PSG_ERR_INTERNAL, "scan not planned in the ingest session");
  auto r = it->second.front();
  it->second.pop_front();
  return std::make_unique<SessionFeed>(*session_, r);
}

// ------------------------------------------------------------------------------ compile
void Execution::compile() {
  plan_.validate();
  shuffle_ = plan_.shuffle_join();
  if (!shuffle_) throw InvalidInput("plans currently require one shuffled join");
  bsrc_ = make_source(plan_, ctx_.footers, shuffle_->build);
  psrc_ = make_source(plan_, ctx_.footers, shuffle_->probe);
  const int bkey = static_cast<int>(bsrc_.wire.require(shuffle_->build_key));
  const int pkey = static_cast<int>(psrc_.wire.require(shuffle_->probe_key));
  if (bsrc_.wire.fields[bkey].type != LType::Int64) throw InvalidInput("partition key must be int64: " + shuffle_->build_key);
  if (psrc_.wire.fields[pkey].type != LType::Int64) throw InvalidInput("partition key must be int64: " + shuffle_->probe_key);
  agg_ = plan_.aggregate.has_value();
  if (agg_) {
    grouped_ = !plan_.aggregate->group_by.empty();
    // joined schema = build payload (wire minus key) ++ probe wire ("_p" on clash)
    Schema joined;
    std::vector<std::pair<int, int>> origin;  // (side, wire idx)
    for (size_t i = 0; i < bsrc_.wire.size(); ++i) {
      if (static_cast<int>(i) == bkey) continue;
      joined.fields.push_back(bsrc_.wire.fields[i]);
      origin.push_back({0, static_cast<int>(i)});
    }
    for (size_t i = 0; i < psrc_.wire.size(); ++i) {
      Field g = psrc_.wire.fields[i];
      if (joined.index_of(g.name)) g.name += "_p";
      joined.fields.push_back(g);
      origin.push_back({1, static_cast<int>(i)});
    }
    if (grouped_) {
      const size_t gi = joined.require(plan_.aggregate->group_by);
      if (origin[gi] != std::make_pair(1, pkey))
        throw InvalidInput("group key resolves to a build payload column; only the probe key is supported");
      result_schema_.fields.push_back(joined.fields[gi]);
    }
    result_schema_.fields.push_back(Field{"rows", LType::Int64});
    for (const auto& c : plan_.aggregate->sums) {
      const size_t si = joined.require(c);
      result_schema_.fields.push_back(Field{"sum_" + joined.fields[si].name, joined.fields[si].type});
      auto [side, w] = origin[si];
      if (side == 1) {
        sum_order.push_back({1, static_cast<int>(probe_sum_wire.size())});
        probe_sum_wire.push_back(w);
      } else {
        sum_order.push_back({0, static_cast<int>(build_sum_wire.size())});
        build_sum_wire.push_back(w);
      }
    }
    if (probe_sum_wire.size() > static_cast<size_t>(kMaxSums) || build_sum_wire.size() > static_cast<size_t>(kMaxSums))
      throw InvalidInput("too many aggregate sums");
  } else {
    for (size_t i = 0; i < bsrc_.wire.size(); ++i)
      if (static_cast<int>(i) != bkey) result_schema_.fields.push_back(bsrc_.wire.fields[i]);
    for (size_t i = 0; i < psrc_.wire.size(); ++i) {
      Field g = psrc_.wire.fields[i];
      if (result_schema_.index_of(g.name)) g.name += "_p";
      result_schema_.fields.push_back(g);
    }
  }
}

ScanProgram Execution::base_program(const SourceDef& s, const RegMap& m, bool with_joins) {
  ScanProgram p;
  std::memset(&p, 0, sizeof p);
  p.n_in = m.n_in;
  p.n_pred = m.n_pred;
  p.n_early = m.n_early;
  p.n_regs = std::max(1, m.n_regs);
  p.n_atoms = static_cast<int>(s.scan->predicate.size());
  if (p.n_atoms > kMaxAtoms) throw InvalidInput("too many predicate atoms");
  for (int a = 0; a < p.n_atoms; ++a) {
    const Atom& at = s.scan->predicate[a];
    const int pi = static_cast<int>(s.proj.schema.require(at.column));
    AtomDesc& d = p.atoms[a];
    d.reg = m.reg_of.at({-1, pi});
    d.op = static_cast<int>(at.op);
    d.is_float = s.proj.schema.fields[pi].type == LType::Float64;
    d.lit = d.is_float ? dbl_bits(at.as_float()) : static_cast<uint64_t>(at.as_int());
  }
  if (with_joins) {
    auto& tables = (&s == &bsrc_) ? bl_tables_ : pl_tables_;
    p.n_joins = static_cast<int>(s.chain.size());
    if (p.n_joins > kMaxJoins) throw InvalidInput("too many local joins");
    for (int j = 0; j < p.n_joins; ++j) {
      JoinDesc& jd = p.joins[j];
      jd.t = tables[j]->dev;
      jd.key_reg = m.reg_of.at(s.stage_refs[j][s.chain[j].probe_key_stage]);
      for (size_t k = 0; k < m.payload_regs[j].size(); ++k) jd.payload_reg[k] = m.payload_regs[j][k];
    }
  }
  p.part_key_reg = -1;
  p.key_reg = -1;
  return p;
}

DevCols Execution::alloc_cols(size_t ncols, uint64_t cap) {
  DevCols c;
  c.cap = cap;
  for (size_t i = 0; i < ncols; ++i) c.cols.emplace_back(ctx_.pool, std::max<uint64_t>(cap, 1) * 8 + 16, ctx_.compute);
  c.count = DevBuf(ctx_.pool, 8, ctx_.compute);
  PSG_CUDA(cudaMemsetAsync(c.count.p, 0, 8, ctx_.compute));
  return c;
}

bool Execution::dup_chain(const SourceDef& s) const {
  const auto& tables = (&s == &bsrc_) ? bl_tables_ : pl_tables_;
  for (const auto& t : tables)
    if (!t->unique) return true;
  return false;
}

DevCols Execution::materialize_chain(const SourceDef& s, const RegMap& m, const BatchView& v,
                                     const std::vector<int>& out_regs) {
  auto& tables = (&s == &bsrc_) ? bl_tables_ : pl_tables_;
  // 1. predicate + compaction of the base columns the chain and the sink read (no joins in-kernel)
  ScanProgram p = base_program(s, m, false);
  std::vector<int> base_regs(m.n_in);
  std::iota(base_regs.begin(), base_regs.end(), 0);
  DevCols base = alloc_cols(base_regs.size(), std::max<uint64_t>(v.rows, 1));
  materialize_into(base, p, v, base_regs, -1, nullptr, false, true);
  uint64_t n = read_count(base);
  std::vector<ColRef> refs;
  for (int c = 0; c < m.n_in; ++c) refs.push_back({-1, m.base_proj[c]});
  std::vector<DevBuf> cols = std::move(base.cols);
  // 2. one expansion per local join, in chain order
  for (size_t j = 0; j < s.chain.size(); ++j) {
    const ColRef kref = s.stage_refs[j][s.chain[j].probe_key_stage];
    const size_t ki = std::find(refs.begin(), refs.end(), kref) - refs.begin();
    if (ki == refs.size()) throw Error(PSG_ERR_INTERNAL, "join key column not materialised");
    const LocalTableDev& t = tables[j]->dev;
    const uint64_t* keys = cols[ki].as<uint64_t>();
    DevBuf counts(ctx_.pool, (n + 1) * 4, ctx_.compute), offs(ctx_.pool, (n + 1) * 4, ctx_.compute);
    PSG_CUDA(cudaMemsetAsync(counts.p, 0, (n + 1) * 4, ctx_.compute));
    launch_expand_count(t, keys, n, counts.as<uint32_t>(), ctx_.compute);
    const size_t tb = exclusive_scan_u32(nullptr, nullptr, n + 1, nullptr, 0, ctx_.compute);
    DevBuf tmp(ctx_.pool, std::max<size_t>(tb, 8), ctx_.compute);
    exclusive_scan_u32(counts.as<uint32_t>(), offs.as<uint32_t>(), n + 1, tmp.p, tb, ctx_.compute);
    uint32_t total = 0;
    PSG_CUDA(cudaMemcpyAsync(&total, offs.as<uint32_t>() + n, 4, cudaMemcpyDeviceToHost, ctx_.compute));
    PSG_CUDA(cudaStreamSynchronize(ctx_.compute));
    const int np = t.npayload;
    std::vector<DevBuf> next;
    std::vector<ColRef> nrefs;
    for (int k = 0; k < np; ++k) {
      next.emplace_back(ctx_.pool, std::max<uint64_t>(total, 1) * 8 + 16, ctx_.compute);
      nrefs.push_back({static_cast<int>(j), m.payload_cols[j][k]});
    }
    for (size_t c = 0; c < cols.size(); ++c) {
      next.emplace_back(ctx_.pool, std::max<uint64_t>(total, 1) * 8 + 16, ctx_.compute);
      nrefs.push_back(refs[c]);
    }
    std::vector<const uint64_t*> in;
    std::vector<uint64_t*> out;
    for (auto& c : cols) in.push_back(c.as<uint64_t>());
    for (auto& c : next) out.push_back(c.as<uint64_t>());
    if (np + in.size() > static_cast<size_t>(kMaxOut)) throw InvalidInput("local join chain carries too many columns");
    launch_expand_write(t, keys, n, offs.as<uint32_t>(), in.data(), static_cast<int>(in.size()), out.data(), ctx_.compute);
    cols = std::move(next);
    refs = std::move(nrefs);
    n = total;
  }
  // 3. the requested registers, in order
  std::map<int, ColRef> ref_of_reg;
  for (const auto& [ref, reg] : m.reg_of) ref_of_reg[reg] = ref;
  DevCols out;
  out.cap = std::max<uint64_t>(n, 1);
  out.rows = n;
  std::vector<bool> taken(cols.size(), false);
  for (int r : out_regs) {
    const size_t i = std::find(refs.begin(), refs.end(), ref_of_reg.at(r)) - refs.begin();
    if (i == refs.size()) throw Error(PSG_ERR_INTERNAL, "chain output column not materialised");
    if (!taken[i]) {
      taken[i] = true;
      out.cols.push_back(std::move(cols[i]));
    } else {  // the same column twice (e.g. key and a sum of it)
      DevBuf cp(ctx_.pool, out.cap * 8 + 16, ctx_.compute);
      PSG_CUDA(cudaMemcpyAsync(cp.p, out.cols[std::find(out_regs.begin(), out_regs.end(), r) - out_regs.begin()].p, n * 8,
                               cudaMemcpyDeviceToDevice, ctx_.compute));
      out.cols.push_back(std::move(cp));
    }
  }
  out.count = DevBuf(ctx_.pool, 8, ctx_.compute);
  PSG_CUDA(cudaMemcpyAsync(out.count.p, &out.rows, 8, cudaMemcpyHostToDevice, ctx_.compute));
  PSG_CUDA(cudaStreamSynchronize(ctx_.compute));  // the host source above is a stack value
  return out;
}

DevCols Execution::concat_cols(std::vector<DevCols>& parts, size_t ncols) {
  uint64_t total = 0;
  for (auto& p : parts) total += p.rows;
  DevCols out = alloc_cols(ncols, std::max<uint64_t>(total, 1));
  uint64_t at = 0;
  for (auto& p : parts) {
    for (size_t c = 0; c < ncols && p.rows; ++c)
      PSG_CUDA(cudaMemcpyAsync(out.cols[c].as<uint64_t>() + at, p.cols[c].p, p.rows * 8, cudaMemcpyDeviceToDevice,
                               ctx_.compute));
    at += p.rows;
  }
  out.rows = total;
  PSG_CUDA(cudaMemcpyAsync(out.count.p, &out.rows, 8, cudaMemcpyHostToDevice, ctx_.compute));
  PSG_CUDA(cudaStreamSynchronize(ctx_.compute));
  parts.clear();
  return out;
}

uint64_t Execution::read_count(DevCols& c) {
  uint64_t n = 0;
  PSG_CUDA(cudaMemcpyAsync(&n, c.count.p, 8, cudaMemcpyDeviceToHost, ctx_.compute));
  PSG_CUDA(cudaStreamSynchronize(ctx_.compute));
  if (n > c.cap) throw Error(PSG_ERR_INTERNAL, "materialisation overflow");
  c.rows = n;
  return n;
}

void Execution::run_scan(const ScanProgram& p, const BatchView& v, bool timed, cudaStream_t stream) {
  if (v.nsegs == 0) return;
  cudaStream_t st = stream ? stream : ctx_.compute;
  std::pair<cudaEvent_t, cudaEvent_t> ev{nullptr, nullptr};
  if (timed) {
    PSG_CUDA(cudaEventCreate(&ev.first));
    PSG_CUDA(cudaEventCreate(&ev.second));
    timed_.push_back(ev);
    PSG_CUDA(cudaEventRecord(ev.first, st));
  }
  fused_scan(p, v.d_segs, v.d_tile_seg, v.nsegs, v.ntiles, st);
  if (timed) {
    PSG_CUDA(cudaEventRecord(ev.second, st));
    st_.probe_kernel_launches += 1;
    st_.probe_kernel_bytes += v.bytes;
  }
}

void Execution::materialize_into(DevCols& out, const ScanProgram& p0, const BatchView& v, const std::vector<int>& out_regs,
                                 int part_key_reg, DevBuf* part_counts, bool timed, bool aligned) {
  ScanProgram p = p0;
  p.sink = SINK_MATERIALIZE;
  p.staged_ok = aligned ? 1 : 0;
  p.n_out = static_cast<int>(out_regs.size());
  for (int o = 0; o < p.n_out; ++o) {
    p.out_reg[o] = out_regs[o];
    p.out_col[o] = out.cols[o].as<uint64_t>();
  }
  p.out_cap = out.cap;
  p.out_count = out.count.as<unsigned long long>();
  if (part_key_reg >= 0 && ctx_.nranks > 1) {
    p.nparts = ctx_.nranks;
    p.part_key_reg = part_key_reg;
    p.part_counts = part_counts->as<unsigned long long>();
  }
  run_scan(p, v, timed);
}

BatchView Execution::upload_segments(std::vector<Segment> segs, DevBuf& holder, cudaStream_t stream) {
  cudaStream_t st = stream ? stream : ctx_.compute;
  BatchView v;
  const uint64_t T = static_cast<uint64_t>(scan_tile_rows());
  uint64_t tiles = 0;
  for (auto& s : segs) {
    s.tile_begin = tiles;
    tiles += (s.rows + T - 1) / T;
    v.rows += s.rows;
  }
  if (segs.empty()) return v;
  size_t toff = 0;
  auto blob = pack_view(segs, toff);
  holder = DevBuf(ctx_.pool, blob.size(), st);
  PSG_CUDA(cudaMemcpyAsync(holder.p, blob.data(), blob.size(), cudaMemcpyHostToDevice, st));
  host_keep_.push_back(std::move(blob));  // pageable source must outlive the async copy
  v.d_segs = holder.as<Segment>();
  v.d_tile_seg = reinterpret_cast<const uint32_t*>(holder.as<uint8_t>() + toff);
  v.nsegs = static_cast<int>(segs.size());
  v.ntiles = tiles;
  return v;
}

// ---------------------------------------------------------------------- local join tables
/// PSG_LOCAL_BITMAP=0 disables the dense semi-join bitmap for local joins (A/B measurements).
static bool bitmap_env() {
  static const bool on = [] {
    const char* e = std::getenv("PSG_LOCAL_BITMAP");
    return !(e && std::string(e) == "0");
  }();
  return on;
}

void Execution::build_local_tables() {
  for (int side = 0; side < 2; ++side) {
    SourceDef& s = side == 0 ? bsrc_ : psrc_;
    auto& tables = side == 0 ? bl_tables_ : pl_tables_;
    for (size_t j = 0; j < s.chain.size(); ++j) {
      LocalJoinDef& lj = s.chain[j];
      auto t = std::make_unique<LocalTable>();
      // program over the replicated scan: predicate + key + needed payload columns
      SourceDef rs;
      rs.scan = lj.scan;
      rs.proj = lj.proj;
      rs.wire = lj.proj.schema;
      std::vector<ColRef> refs;
      for (size_t i = 0; i < rs.wire.size(); ++i) refs.push_back({-1, static_cast<int>(i)});
      rs.stage_refs.push_back(refs);
      // needed payload of this join = payload cols referenced by the consuming programs; we load
      // every payload column the source may need (computed by the caller's RegMap later), so
      // conservatively take all payload columns that appear in any needed ref.
      std::vector<int> needed{lj.key_idx};
      for (int p : lj.needed_payload) needed.push_back(lj.payload_idx[p]);
      RegMap m = analyse(rs, needed, -1, false);
      ScanProgram p = base_program(rs, m, false);
      std::vector<int> out_regs;
      for (int w : needed) out_regs.push_back(m.reg_of.at({-1, w}));
      PSG_TRACE_MSG("local table %s: regs %d in %d", lj.node->id.c_str(), m.n_regs, m.n_in);
      auto feed = open_feed(*rs.scan, file_cols_of(rs, m));
      PSG_TRACE_MSG("local table: feed %zu batches %llu rows", feed->nbatches, static_cast<unsigned long long>(feed->total_rows));
      // Semi-join build straight into the membership bitmap (no payload, unique keys): the scan
      // sets each surviving key's bit (SINK_KEYBITS) - no materialised keys, no bitmap pass. A
      // duplicate key (or one outside the zone-map range) re-runs the query on the CSR table path.
      if (lj.needed_payload.empty() && bitmap_env() && keybits_env() && jit_available() && !ctx_.no_keybits) {
        long long lohi[2] = {LLONG_MAX, LLONG_MIN};
        zone_range(lj.scan->paths, lj.proj.file_idx[lj.key_idx], lohi[0], lohi[1]);
        const uint64_t range = lohi[1] >= lohi[0] ? static_cast<uint64_t>(lohi[1]) - static_cast<uint64_t>(lohi[0]) + 1 : 0;
        if (range != 0 && range <= (1ULL << 34) && range / 64 <= feed->total_rows) {
          const uint64_t words = (range + 31) / 32;
          t->bitmap = DevBuf(ctx_.pool, words * 4, ctx_.compute);
          DevBuf kc(ctx_.pool, 16, ctx_.compute);
          PSG_CUDA(cudaMemsetAsync(t->bitmap.p, 0, words * 4, ctx_.compute));
          PSG_CUDA(cudaMemsetAsync(kc.p, 0, 16, ctx_.compute));
          ScanProgram kp = p;
          kp.sink = SINK_KEYBITS;
          kp.staged_ok = 1;
          kp.key_reg = out_regs[0];
          kp.kb_bits = t->bitmap.as<uint32_t>();
          kp.kb_min = lohi[0];
          kp.kb_range = range;
          kp.kb_count = kc.as<unsigned long long>();
          kp.kb_flag = reinterpret_cast<unsigned int*>(kc.as<unsigned long long>() + 1);
          BatchView v;
          while (feed->next(v)) {
            run_scan(kp, v, false);
            feed->done();
            st_.ingest_bytes += v.bytes;
          }
          // optimistic: the duplicate flag is read with the query's next host read (check_lt_flags;
          // no sync here). Duplicates re-run the query with the materialising build (the
          // replicated scan is the same on every rank, so every rank decides alike).
          lt_flags_.push_back(std::move(kc));
          t->unique = true;
          std::memset(&t->dev, 0, sizeof t->dev);
          t->dev.bitmap = t->bitmap.as<uint32_t>();
          t->dev.bmin = lohi[0];
          t->dev.brange = range;
          tables.push_back(std::move(t));
          continue;
        }
      }
      DevCols mat = alloc_cols(out_regs.size(), std::max<uint64_t>(feed->total_rows, 1));
      BatchView v;
      while (feed->next(v)) {
        materialize_into(mat, p, v, out_regs, -1, nullptr, false, true);
        feed->done();
        st_.ingest_bytes += v.bytes;
      }
      const uint64_t n = read_count(mat);
      const int np = static_cast<int>(lj.needed_payload.size());
      // Semi-join fast path: no payload needed and the keys are unique and dense -> a membership
      // bitmap over [min, max] (Q3's 3 M customer keys in 15 M: 1.9 MB, L2-resident) replaces the
      // hash table; probes become one cached bit test.
      if (np == 0 && n > 0 && bitmap_env()) {
        // key range from the replicated scan's footer zone maps (a superset of the surviving keys)
        long long lohi[2] = {LLONG_MAX, LLONG_MIN};
        zone_range(lj.scan->paths, lj.proj.file_idx[lj.key_idx], lohi[0], lohi[1]);
        const uint64_t range = static_cast<uint64_t>(lohi[1]) - static_cast<uint64_t>(lohi[0]) + 1;
        if (range != 0 && range <= (1ULL << 34) && range / 64 <= n) {
          const uint64_t words = (range + 31) / 32;
          t->bitmap = DevBuf(ctx_.pool, words * 4, ctx_.compute);
          DevBuf dup(ctx_.pool, 4, ctx_.compute);
          PSG_CUDA(cudaMemsetAsync(t->bitmap.p, 0, words * 4, ctx_.compute));
          PSG_CUDA(cudaMemsetAsync(dup.p, 0, 4, ctx_.compute));
          launch_bitmap_set(mat.cols[0].as<uint64_t>(), n, lohi[0], t->bitmap.as<uint32_t>(), dup.as<unsigned int>(),
                            ctx_.compute);
          unsigned int d = 0;
          PSG_CUDA(cudaMemcpyAsync(&d, dup.p, 4, cudaMemcpyDeviceToHost, ctx_.compute));
          PSG_CUDA(cudaStreamSynchronize(ctx_.compute));
          if (!d) {  // unique: bitmap mode
            t->unique = true;
            std::memset(&t->dev, 0, sizeof t->dev);
            t->dev.bitmap = t->bitmap.as<uint32_t>();
            t->dev.bmin = lohi[0];
            t->dev.brange = range;
            tables.push_back(std::move(t));
            continue;
          }
          t->bitmap.reset();
        }
      }
      // CSR hash table
      t->cap = pow2_at_least(std::max<uint64_t>(2 * n, 16));
      t->keys = DevBuf(ctx_.pool, t->cap * 8, ctx_.compute);
      t->cnt = DevBuf(ctx_.pool, (t->cap + 1) * 4, ctx_.compute);
      t->start = DevBuf(ctx_.pool, (t->cap + 1) * 4, ctx_.compute);
      DevBuf cursor(ctx_.pool, (t->cap + 1) * 4, ctx_.compute);
      DevBuf maxc(ctx_.pool, 4, ctx_.compute);
      PSG_CUDA(cudaMemsetAsync(maxc.p, 0, 4, ctx_.compute));
      PSG_CUDA(cudaMemsetAsync(cursor.p, 0, (t->cap + 1) * 4, ctx_.compute));
      launch_local_init(t->keys.as<uint64_t>(), t->cnt.as<uint32_t>(), t->cap, ctx_.compute);
      const uint64_t* bk = mat.cols[0].as<uint64_t>();
      launch_local_count(t->keys.as<uint64_t>(), t->cnt.as<uint32_t>(), t->cap - 1, shift_of(t->cap), bk, n, maxc.as<unsigned>(),
                         ctx_.compute);
      size_t tb = exclusive_scan_u32(nullptr, nullptr, t->cap + 1, nullptr, 0, ctx_.compute);
      DevBuf tmp(ctx_.pool, tb, ctx_.compute);
      exclusive_scan_u32(t->cnt.as<uint32_t>(), t->start.as<uint32_t>(), t->cap + 1, tmp.p, tb, ctx_.compute);
      std::vector<const uint64_t*> src;
      std::vector<uint64_t*> dst;
      for (int k = 0; k < np; ++k) {
        t->payload.emplace_back(ctx_.pool, std::max<uint64_t>(n, 1) * 8, ctx_.compute);
        src.push_back(mat.cols[1 + k].as<uint64_t>());
        dst.push_back(t->payload.back().as<uint64_t>());
      }
      launch_local_fill(t->keys.as<uint64_t>(), t->start.as<uint32_t>(), cursor.as<uint32_t>(), t->cap - 1, shift_of(t->cap), bk,
                        src.data(),
                        dst.data(), np, n, ctx_.compute);
      unsigned mx = 0;
      PSG_CUDA(cudaMemcpyAsync(&mx, maxc.p, 4, cudaMemcpyDeviceToHost, ctx_.compute));
      PSG_CUDA(cudaStreamSynchronize(ctx_.compute));
      t->unique = mx <= 1;
      t->dev.keys = t->keys.as<uint64_t>();
      t->dev.cnt = t->cnt.as<uint32_t>();
      t->dev.start = t->start.as<uint32_t>();
      t->dev.mask = t->cap - 1;
      t->dev.shift = shift_of(t->cap);
      t->dev.npayload = np;
      for (int k = 0; k < np; ++k) t->dev.payload[k] = t->payload[k].as<uint64_t>();
      tables.push_back(std::move(t));
    }
  }
}

// --------------------------------------------------------------------------- agg table
void Execution::build_agg_table(uint64_t build_rows, uint64_t bloom_words, uint64_t rank_slots) {
  // rank_slots > 0: rank-indexed table of exactly that many slots (+ the spill slot), written
  // whole by the rank build (no init pass, no hashing)
  agg_cap_ = rank_slots ? rank_slots : pow2_at_least(std::max<uint64_t>(2 * build_rows, 16));
  const int nps = static_cast<int>(probe_sum_wire.size()), nbs = static_cast<int>(build_sum_wire.size());
  int hw = 2 + nps;
  hw = hw <= 2 ? 2 : (hw <= 4 ? 4 : 8 * ((hw + 7) / 8));
  const int cw = rank_slots ? (4 + nbs) & ~3 : 1 + nbs;  // rank table: whole 32-byte rows
  agg_hot_ = DevBuf(ctx_.pool, (agg_cap_ + 1) * hw * 8, ctx_.compute);
  agg_cold_ = DevBuf(ctx_.pool, (agg_cap_ + 1) * cw * 8, ctx_.compute);
  std::memset(&aggt_, 0, sizeof aggt_);
  aggt_.hot = agg_hot_.as<uint64_t>();
  aggt_.cold = agg_cold_.as<uint64_t>();
  aggt_.mask = agg_cap_ - 1;
  aggt_.shift = rank_slots ? 0 : shift_of(agg_cap_);
  aggt_.hw = hw;
  aggt_.cw = cw;
  aggt_.nps = nps;
  aggt_.nbs = nbs;
  for (int i = 0; i < nps; ++i) aggt_.ps_float[i] = psrc_.wire.fields[probe_sum_wire[i]].type == LType::Float64;
  for (int i = 0; i < nbs; ++i) aggt_.bs_float[i] = bsrc_.wire.fields[build_sum_wire[i]].type == LType::Float64;
  agg_dups_ = DevBuf(ctx_.pool, 4, ctx_.compute);
  PSG_CUDA(cudaMemsetAsync(agg_dups_.p, 0, 4, ctx_.compute));
  aggt_.dups = agg_dups_.as<unsigned int>();
  if (bloom_words) {
    agg_bloom_ = DevBuf(ctx_.pool, bloom_words * 4, ctx_.compute);
    aggt_.bloom = agg_bloom_.as<uint32_t>();
    aggt_.bloom_mask = bloom_words - 1;
    aggt_.bloom_shift = shift_of(bloom_words);
  }
  if (!rank_slots) launch_agg_init(aggt_, agg_cap_, ctx_.compute);
}

/// Bucketed aggregation for the one-GPU rank-indexed table (ScanProgram::bkt, k_bucket_agg):
/// possible when every probe-side sum is an int column of the probe scan whose zone-map span fits,
/// with the slot's low bits, in one 64-bit word. Bucket capacity: the expected survivors (probe
/// rows x the build keys' share of the key range) / buckets x 1.5; overflow is applied directly.
/// PSG_BUCKETS=0: off.
bool Execution::setup_buckets(const int64_t* prange_lo, const int64_t* prange_hi, uint64_t probe_rows_all) {
  static const bool env = [] {
    const char* e = std::getenv("PSG_BUCKETS");
    return !(e && e[0] == '0');
  }();
  const int np = static_cast<int>(probe_sum_wire.size());
  if (!env || ctx_.no_buckets || !jit_available() || np > 3 || aggt_.krange == 0 || agg_cap_ == 0) return false;
  BucketDev bd{};
  int shift = kBucketBits;
  uint64_t probe_rows = probe_rows_all;
  if (!probe_rows)
    for (const auto& path : psrc_.scan->paths) probe_rows += ctx_.footers.get(path)->total_rows();
  for (int k = 0; k < np; ++k) {
    const ColRef ref = psrc_.stage_refs.back()[probe_sum_wire[k]];
    if (ref.join >= 0 || psrc_.wire.fields[probe_sum_wire[k]].type != LType::Int64) return false;
    long long lo = LLONG_MAX, hi = LLONG_MIN;
    if (prange_lo)
      lo = prange_lo[k], hi = prange_hi[k];
    else
      zone_range(psrc_.scan->paths, psrc_.proj.file_idx[ref.idx], lo, hi);
    if (hi < lo) lo = hi = 0;
    const uint64_t span = static_cast<uint64_t>(hi) - static_cast<uint64_t>(lo);
    const int w = span ? 64 - __builtin_clzll(span) : 0;
    if (shift + w > 64) return false;
    bd.shift[k] = shift;
    bd.mask[k] = w == 64 ? ~0ULL : ((1ULL << w) - 1);
    bd.min[k] = lo;
    bd.word[k] = 1 + k;  // hot word 2 + k
    shift += w;
  }
  const uint64_t nb = (agg_cap_ + kBucketSlots - 1) / kBucketSlots;
  const double share = std::min(1.0, static_cast<double>(agg_cap_) / static_cast<double>(aggt_.krange));
  // PSG_BUCKET_CAP / PSG_BUCKET_OVF_CAP override the capacities (tests: force the overflow paths)
  static const uint64_t cap_env = [] {
    const char* e = std::getenv("PSG_BUCKET_CAP");
    return e ? std::strtoull(e, nullptr, 10) : 0ULL;
  }();
  // 2^sub_bits sub-lists per bucket (PSG_BUCKET_SUB): more distinct append counters. SF100 A/B:
  // one GPU 4.60 ms with 1 sub-list vs 4.79 with 16 (the emit walks 16 lists, the probe keeps 16x
  // more open bucket tails); N=2 4.15 vs 4.07 (the owner-side fold of the received rows, a burst
  // of appends, 0.43 -> 0.20 ms); at N=2 4 sub-lists measured best (query 3.31 / 3.21 / 3.29 /
  // 3.29 ms for 1 / 4 / 8 / 16). Default: 1 at one GPU, 4 at N > 1.
  static const int sub_env = [] {
    const char* e = std::getenv("PSG_BUCKET_SUB");
    return e ? std::max(1, std::atoi(e)) : 0;
  }();
  const int sub_req = sub_env ? sub_env : (ctx_.nranks > 1 ? 4 : 1);
  int sub_bits = 0;
  while ((2 << sub_bits) <= sub_req && sub_bits < 5) ++sub_bits;
  const uint64_t nsub = nb << sub_bits;
  const uint64_t cap = cap_env ? cap_env
                               : static_cast<uint64_t>(1.5 * static_cast<double>(probe_rows) * share / static_cast<double>(nsub)) +
                                     (1024 >> sub_bits) + 64;
  if (cap >= (1ULL << 31)) return false;
  bkt_ = DevBuf(ctx_.pool, nsub * cap * 8, ctx_.compute);
  bkt_fill_ = DevBuf(ctx_.pool, nsub * 4, ctx_.compute);
  PSG_CUDA(cudaMemsetAsync(bkt_fill_.p, 0, nsub * 4, ctx_.compute));
  bd.bkt = bkt_.as<uint64_t>();
  bd.fill = bkt_fill_.as<unsigned int>();
  bd.cap = static_cast<uint32_t>(cap);
  bd.sub_bits = sub_bits;
  bd.nacc = 1 + np;
  static const uint32_t kOvfCap = [] {  // 1 MB: scanned by every bucket CTA when not empty
    const char* e = std::getenv("PSG_BUCKET_OVF_CAP");
    return e ? static_cast<uint32_t>(std::strtoul(e, nullptr, 10)) : (1u << 16);
  }();
  bkt_ovf_ = DevBuf(ctx_.pool, kOvfCap * 16, ctx_.compute);
  bkt_ovf_count_ = DevBuf(ctx_.pool, 4, ctx_.compute);
  PSG_CUDA(cudaMemsetAsync(bkt_ovf_count_.p, 0, 4, ctx_.compute));
  bd.ovf = bkt_ovf_.as<uint64_t>();
  bd.ovf_count = bkt_ovf_count_.as<unsigned int>();
  bd.ovf_cap = kOvfCap;
  bd_ = bd;
  nbuckets_ = nb;
  return true;
}

void Execution::apply_buckets(ScanProgram& p) const {
  p.bkt_ovf = const_cast<uint64_t*>(bd_.ovf);
  p.bkt_ovf_count = const_cast<unsigned int*>(bd_.ovf_count);
  p.bkt_ovf_cap = bd_.ovf_cap;
  p.bkt = const_cast<uint64_t*>(bd_.bkt);
  p.bkt_fill = const_cast<unsigned int*>(bd_.fill);
  p.bkt_cap = bd_.cap;
  p.bkt_sub_bits = bd_.sub_bits;
  for (int k = 0; k < kMaxSums; ++k) {
    p.bkt_shift[k] = bd_.shift[k];
    p.bkt_mask[k] = bd_.mask[k];
    p.bkt_min[k] = bd_.min[k];
  }
}

/// Bucketed finalisation: one kernel folds every bucket, finds its output offset by decoupled
/// look-back and writes its rows in key order (k_bucket_emit); the group total (the last bucket's
/// inclusive prefix) is read once at the end, when the rows go to the host.
void Execution::finalize_buckets(ResultRows& out, bool want_rows) {
  const int nc = static_cast<int>(result_schema_.size());
  std::vector<int32_t> kind, idx;
  kind.push_back(0), idx.push_back(0);
  kind.push_back(1), idx.push_back(0);
  for (auto [side, k] : sum_order) {
    kind.push_back(side == 1 ? 2 : 3);
    idx.push_back(k);
  }
  // rows are written at their final offsets: size the output for the upper bound (one group per
  // build key) instead of syncing on the count
  DevBuf state(ctx_.pool, nbuckets_ * 8, ctx_.compute), ticket(ctx_.pool, 8, ctx_.compute);
  DevBuf first_word(ctx_.pool, nbuckets_ * 4, ctx_.compute);
  DevBuf rows(ctx_.pool, std::max<uint64_t>(agg_cap_, 1) * nc * 8, ctx_.compute);
  launch_bucket_emit(aggt_, bd_, nbuckets_, agg_cap_, state.as<unsigned long long>(), ticket.as<unsigned int>(),
                     first_word.as<uint32_t>(), nc, kind.data(), idx.data(), rows.as<uint64_t>(), ctx_.compute);
  DevBuf o;
  const void* ovf = bd_.ovf_count;
  if (ctx_.nranks > 1) {  // the re-run decision is collective: the largest overflow of any rank
    o = DevBuf(ctx_.pool, 4, ctx_.compute);
    PSG_NCCL(ncclAllReduce(bd_.ovf_count, o.p, 1, ncclUint32, ncclMax, ctx_.nccl, ctx_.compute));
    ovf = o.p;
  }
  uint64_t w[3] = {0, 0, 0};
  const void* last_p = state.as<unsigned long long>() + (nbuckets_ - 1);
  if (slab_recv_.p) read_words({{last_p, false}, {ovf, true}, {slab_recv_.p, false}}, w);
  else read_words({{last_p, false}, {ovf, true}}, w);
  const unsigned long long last = w[0], recv = w[2];
  const uint64_t novf = w[1];
  st_.bucket_overflow = novf;
  if (slab_recv_.p) {
    st_.bytes_received += recv * 8;
    st_.shuffle_fused = 1;
  }
  if (novf > bd_.ovf_cap) throw BucketOverflow();  // execute_plan re-runs the query without buckets
  const uint64_t ng = last & ((1ULL << 62) - 1);
  out.nrows = ng;
  if (want_rows) {
    uint64_t* dst = out.mutable_rows(ng * nc);
    if (ng) PSG_CUDA(cudaMemcpyAsync(dst, rows.p, ng * nc * 8, cudaMemcpyDeviceToHost, ctx_.compute));
    st_.result_bytes += ng * nc * 8;
  }
  PSG_CUDA(cudaStreamSynchronize(ctx_.compute));
}

/// Bit-packed accumulators: the footer zone maps bound every int probe-side sum column and the
/// total probe row count bounds any group's hits, so the hit count and each sum whose field
/// (offset by its minimum) provably fits share word 1 of the hot slot - one atomicAdd per matched
/// row instead of one per accumulator (Q3: hits + discount in one word, price alone: 2 instead
/// of 3). Bounds are all-reduced at N > 1 (a rank's table also receives other ranks' rows).
/// PSG_ACCPACK=0: off.
void Execution::pack_accumulators() {
  static const bool env = [] {
    const char* e = std::getenv("PSG_ACCPACK");
    return !(e && std::string(e) == "0");
  }();
  if (!env || !grouped_ || !jit_available() || ctx_.p2p) return;
  const int np = static_cast<int>(probe_sum_wire.size());
  if (np == 0) return;
  // [~min_0..np), max_0..np), rows] all-reduced with MAX (rows as MAX of the SUM-encoded... SUM below)
  std::vector<long long> mm(2 * np, 0);
  long long rows = 0;
  std::vector<bool> ok(np, true);
  for (const auto& path : psrc_.scan->paths) rows += static_cast<long long>(ctx_.footers.get(path)->total_rows());
  for (int k = 0; k < np; ++k) {
    long long lo = LLONG_MAX, hi = LLONG_MIN;
    const ColRef ref = psrc_.stage_refs.back()[probe_sum_wire[k]];
    if (ref.join >= 0 || psrc_.wire.fields[probe_sum_wire[k]].type != LType::Int64) {
      lo = LLONG_MIN, hi = LLONG_MAX;
    } else {
      zone_range(psrc_.scan->paths, psrc_.proj.file_idx[ref.idx], lo, hi);
    }
    mm[k] = ~lo;
    mm[np + k] = hi;
  }
  if (ctx_.nranks > 1) {
    DevBuf d(ctx_.pool, (2 * np + 1) * 8, ctx_.compute);
    PSG_CUDA(cudaMemcpyAsync(d.p, mm.data(), 2 * np * 8, cudaMemcpyHostToDevice, ctx_.compute));
    PSG_CUDA(cudaMemcpyAsync(d.as<long long>() + 2 * np, &rows, 8, cudaMemcpyHostToDevice, ctx_.compute));
    PSG_NCCL(ncclAllReduce(d.p, d.p, 2 * np, ncclInt64, ncclMax, ctx_.nccl, ctx_.compute));
    PSG_NCCL(ncclAllReduce(d.as<long long>() + 2 * np, d.as<long long>() + 2 * np, 1, ncclInt64, ncclSum, ctx_.nccl,
                           ctx_.compute));
    PSG_CUDA(cudaMemcpyAsync(mm.data(), d.p, 2 * np * 8, cudaMemcpyDeviceToHost, ctx_.compute));
    PSG_CUDA(cudaMemcpyAsync(&rows, d.as<long long>() + 2 * np, 8, cudaMemcpyDeviceToHost, ctx_.compute));
    PSG_CUDA(cudaStreamSynchronize(ctx_.compute));
  }
  auto bits = [](unsigned __int128 x) {
    int b = 0;
    while (x) ++b, x >>= 1;
    return b;
  };
  const int bh = bits(static_cast<unsigned __int128>(std::max<long long>(rows, 1)));
  int shift = bh, packed = 0;
  for (int k = 0; k < np; ++k) {
    aggt_.packed_shift[k] = -1;
    const long long lo = ~mm[k], hi = mm[np + k];
    if (aggt_.ps_float[k] || hi < lo || lo == LLONG_MIN || hi == LLONG_MAX) continue;
    const unsigned __int128 span = static_cast<unsigned __int128>(static_cast<uint64_t>(hi) - static_cast<uint64_t>(lo));
    const int b = bits(span * static_cast<unsigned __int128>(rows));
    if (b > 63 || shift + b > 64) continue;
    aggt_.packed_shift[k] = shift;
    aggt_.packed_mask[k] = b == 0 ? 0 : (b == 64 ? ~0ULL : ((1ULL << b) - 1));
    aggt_.packed_min[k] = lo;
    shift += b;
    ++packed;
  }
  if (packed) {
    aggt_.npacked = packed;
    aggt_.hits_mask = bh >= 64 ? ~0ULL : ((1ULL << bh) - 1);
  }
}

/// Same layout as build_agg_table but carved from the symmetric heap with a capacity every rank
/// derives from the same (all-reduced) maximum, so offsets match across ranks.
bool Execution::build_symmetric_agg_table(uint64_t max_rows, bool bloom) {
  agg_cap_ = pow2_at_least(std::max<uint64_t>(2 * max_rows, 16));
  const int nps = static_cast<int>(probe_sum_wire.size()), nbs = static_cast<int>(build_sum_wire.size());
  int hw = 2 + nps;
  hw = hw <= 2 ? 2 : (hw <= 4 ? 4 : 8 * ((hw + 7) / 8));
  const int cw = 1 + nbs;
  const uint64_t words = bloom ? std::min<uint64_t>(pow2_at_least(std::max<uint64_t>(max_rows / 2, 1024)), 8ull << 20) : 0;
  uint8_t* hot = ctx_.symm_alloc((agg_cap_ + 1) * hw * 8);
  uint8_t* cold = ctx_.symm_alloc((agg_cap_ + 1) * cw * 8);
  uint8_t* bl = words ? ctx_.symm_alloc(words * 4) : nullptr;
  if (!hot || !cold || (words && !bl)) return false;
  std::memset(&aggt_, 0, sizeof aggt_);
  aggt_.hot = reinterpret_cast<uint64_t*>(hot);
  aggt_.cold = reinterpret_cast<uint64_t*>(cold);
  aggt_.mask = agg_cap_ - 1;
  aggt_.shift = shift_of(agg_cap_);
  aggt_.hw = hw;
  aggt_.cw = cw;
  aggt_.nps = nps;
  aggt_.nbs = nbs;
  for (int i = 0; i < nps; ++i) aggt_.ps_float[i] = psrc_.wire.fields[probe_sum_wire[i]].type == LType::Float64;
  for (int i = 0; i < nbs; ++i) aggt_.bs_float[i] = bsrc_.wire.fields[build_sum_wire[i]].type == LType::Float64;
  if (words) {
    aggt_.bloom = reinterpret_cast<uint32_t*>(bl);
    aggt_.bloom_mask = words - 1;
    aggt_.bloom_shift = shift_of(words);
  }
  launch_agg_init(aggt_, agg_cap_, ctx_.compute);
  return true;
}

bool Execution::ensure_symmetric(size_t bytes) {
  bytes += Ctx::kSymmReserve;
  if (ctx_.symm_bytes >= bytes) return true;
  if (ctx_.symm_failed) return false;
  // collective: grow every rank's heap together (1 GiB granules), re-mapping the peers' heaps
  ctx_.free_symmetric_heap();
  ctx_.init_symmetric_heap((bytes + (1ull << 30) - 1) & ~((1ull << 30) - 1));
  if (ctx_.symm_bytes == 0) ctx_.symm_failed = true;  // (all ranks voted alike)
  return ctx_.symm_bytes >= bytes;
}

/// Device-side barrier across ranks: a one-word all-reduce on the compute stream completes only
/// after every rank's preceding kernels (including their peer-memory writes) have finished.
void Execution::gpu_barrier() {
  // with the symmetric heap mapped (every rank alike): flag stores through NVLink, no NCCL launch.
  // PSG_PEER_BARRIER=0: the one-word all-reduce.
  static const bool peer_env = [] {
    const char* e = std::getenv("PSG_PEER_BARRIER");
    return !(e && e[0] == '0');
  }();
  if (peer_env && ctx_.symm_bytes > 0 && ctx_.nranks <= kMaxSlabPeers) {
    if (!barrier_err_.p) {
      barrier_err_ = DevBuf(ctx_.pool, 4, ctx_.compute);
      PSG_CUDA(cudaMemsetAsync(barrier_err_.p, 0, 4, ctx_.compute));
    }
    PeerFlags f{};
    for (int r = 0; r < ctx_.nranks; ++r) f.flag[r] = ctx_.barrier_flags(r);
    launch_peer_barrier(f, ctx_.barrier_flags(ctx_.rank), ctx_.rank, ctx_.nranks, ++ctx_.barrier_epoch,
                        barrier_err_.as<unsigned int>(), ctx_.compute);
    return;
  }
  if (!barrier_word_.p) {
    barrier_word_ = DevBuf(ctx_.pool, 8, ctx_.compute);
    PSG_CUDA(cudaMemsetAsync(barrier_word_.p, 0, 8, ctx_.compute));
  }
  PSG_NCCL(ncclAllReduce(barrier_word_.p, barrier_word_.p, 1, ncclUint64, ncclMax, ctx_.nccl, ctx_.compute));
}

// ---------------------------------------------------------------------------- shuffle
Execution::Received Execution::exchange(DevCols& mat, int ncols, int key_col, DevBuf& part_counts, bool have_data,
                                        KeyField kf, cudaStream_t stream) {
  cudaStream_t st = stream ? stream : ctx_.compute;
  const int n = ctx_.nranks;
  Received rcv;
  const int tl = ctx_.timeline ? ctx_.timeline->gpu_begin("exchange w" + std::to_string(st_.waves), 4, st) : -1;
  // dest bases (exclusive scan of the per-destination histogram) and scatter into send regions
  DevBuf base(ctx_.pool, n * 8, st), cursor(ctx_.pool, n * 8, st);
  size_t tb = exclusive_scan_u64(nullptr, nullptr, n, nullptr, 0, st);
  DevBuf tmp(ctx_.pool, tb, st);
  exclusive_scan_u64(part_counts.as<unsigned long long>(), base.as<unsigned long long>(), n, tmp.p, tb, st);
  PSG_CUDA(cudaMemsetAsync(cursor.p, 0, n * 8, st));
  // counts matrix: allgather of every rank's histogram
  DevBuf matrix(ctx_.pool, static_cast<size_t>(n) * n * 8, st);
  PSG_NCCL(ncclAllGather(part_counts.p, matrix.p, n, ncclUint64, ctx_.nccl, st));
  std::vector<uint64_t> m(static_cast<size_t>(n) * n);
  PSG_CUDA(cudaMemcpyAsync(m.data(), matrix.p, m.size() * 8, cudaMemcpyDeviceToHost, st));
  PSG_CUDA(cudaStreamSynchronize(st));  // the one data-dependent host sync per wave
  PhaseTimer xt;
  const int me = ctx_.rank;
  const ExchangePlan xp = plan_exchange(m.data(), n, me);
  const uint64_t nrows = xp.send_rows;
  DevBuf send(ctx_.pool, std::max<uint64_t>(nrows, 1) * ncols * 8, st);
  if (have_data && nrows) {
    std::vector<const uint64_t*> in;
    for (int c = 0; c < ncols; ++c) in.push_back(mat.cols[c].as<uint64_t>());
    launch_part_scatter(in.data(), ncols, nrows, key_col, n, base.as<unsigned long long>(),
                        part_counts.as<unsigned long long>(), cursor.as<unsigned long long>(), send.as<uint64_t>(),
                        st, kf);
  }
  const uint64_t rtotal = xp.recv_rows;
  rcv.buf = DevBuf(ctx_.pool, std::max<uint64_t>(rtotal, 1) * ncols * 8 + 16, st);
  rcv.rows = rtotal;
  xfer_ev_.push_back(std::make_unique<TimedPair>());
  PSG_CUDA(cudaEventRecord(xfer_ev_.back()->a, st));
  PSG_NCCL(ncclGroupStart());
  for (int p = 0; p < n; ++p) {
    const uint64_t sc = xp.send_cnt[p], rc = xp.recv_cnt[p];
    const uint64_t soff = xp.send_off[p], roff = xp.recv_off[p];
    if (sc) PSG_NCCL(ncclSend(send.as<uint64_t>() + soff * ncols, sc * ncols, ncclUint64, p, ctx_.nccl, st));
    if (rc) PSG_NCCL(ncclRecv(rcv.buf.as<uint64_t>() + roff * ncols, rc * ncols, ncclUint64, p, ctx_.nccl, st));
    if (rc) {
      Segment sg;
      std::memset(&sg, 0, sizeof sg);
      for (int c = 0; c < ncols; ++c) sg.col[c] = rcv.buf.as<uint64_t>() + roff * ncols + c * rc;
      sg.rows = rc;
      rcv.segs.push_back(sg);
      if (p != me) st_.bytes_received += rc * ncols * 8;
    }
    if (p != me) st_.bytes_sent += sc * ncols * 8;
  }
  PSG_NCCL(ncclGroupEnd());
  PSG_CUDA(cudaEventRecord(xfer_ev_.back()->b, st));
  if (tl >= 0) ctx_.timeline->gpu_end(tl, st);
  xt.mark("  exchange payload", st);
  st_.waves += 1;
  return rcv;
}

// ---------------------------------------------------------------------------- finalize
/// Result rows in signed key order (HashAggregator's std::map order, pipeline.cpp:296-305).
/// Dense keys (range <= 256 x groups, e.g. order keys): the output position of a group is its
/// key's rank in a bitmap of present keys, so one sequential table pass writes every row in
/// place (no sort, no gather). Sparse keys: compact -> radix sort of the varying key bits -> emit.
void Execution::finalize_grouped(ResultRows& out, bool want_rows) {
  if (bucket_mode_) return finalize_buckets(out, want_rows);
  const uint64_t nslots = agg_cap_ + 1;
  DevBuf counter(ctx_.pool, 24, ctx_.compute);
  const uint64_t init[3] = {0, ~0ULL, 0};
  uint64_t cnt[3] = {0, 0, 0};
  static const bool dense_env = [] {
    const char* e = std::getenv("PSG_DENSE_EMIT");
    return !(e && std::string(e) == "0");
  }();
  const uint64_t flip = 0x8000000000000000ULL;
  if (aggt_.kbits != nullptr && dense_env) {
    // the exact build-key range bounds every group: no range pass; the group count comes out of
    // the bitmap prefix below
    cnt[0] = ~0ULL;
    cnt[1] = static_cast<uint64_t>(aggt_.kmin) ^ flip;
    cnt[2] = (static_cast<uint64_t>(aggt_.kmin) + aggt_.krange - 1) ^ flip;
  } else {
    PSG_CUDA(cudaMemcpyAsync(counter.p, init, 24, cudaMemcpyHostToDevice, ctx_.compute));
    launch_agg_range(aggt_, agg_cap_, counter.as<unsigned long long>(), ctx_.compute);
    PSG_CUDA(cudaMemcpyAsync(cnt, counter.p, 24, cudaMemcpyDeviceToHost, ctx_.compute));
    PSG_CUDA(cudaStreamSynchronize(ctx_.compute));
  }
  uint64_t ng = cnt[0];
  const int nc = static_cast<int>(result_schema_.size());
  std::vector<int32_t> kind, idx;
  kind.push_back(0), idx.push_back(0);
  kind.push_back(1), idx.push_back(0);
  for (auto [side, k] : sum_order) {
    kind.push_back(side == 1 ? 2 : 3);
    idx.push_back(k);
  }
  DevBuf rows;
  const uint64_t span = ng ? cnt[2] - cnt[1] : 0;  // flipped-key range - 1
  const bool known = ng != ~0ULL;
  if (ng && dense_env && span < (1ULL << 36) && (!known || span / 64 + 1 <= 4 * ng)) {
    const uint64_t words = span / 64 + 1;
    DevBuf bitmap(ctx_.pool, words * 8, ctx_.compute), pc(ctx_.pool, words * 4, ctx_.compute),
        prefix(ctx_.pool, words * 4, ctx_.compute);
    PSG_CUDA(cudaMemsetAsync(bitmap.p, 0, words * 8, ctx_.compute));
    launch_agg_mark(aggt_, agg_cap_, cnt[1], bitmap.as<unsigned long long>(), ctx_.compute);
    launch_popc64(bitmap.as<unsigned long long>(), words, pc.as<uint32_t>(), ctx_.compute);
    const size_t tb = exclusive_scan_u32(nullptr, nullptr, words, nullptr, 0, ctx_.compute);
    DevBuf tmp(ctx_.pool, std::max<size_t>(tb, 8), ctx_.compute);
    exclusive_scan_u32(pc.as<uint32_t>(), prefix.as<uint32_t>(), words, tmp.p, tb, ctx_.compute);
    if (!known) {  // groups = last prefix + last count
      uint32_t tail[2] = {0, 0};
      PSG_CUDA(cudaMemcpyAsync(&tail[0], prefix.as<uint32_t>() + words - 1, 4, cudaMemcpyDeviceToHost, ctx_.compute));
      PSG_CUDA(cudaMemcpyAsync(&tail[1], pc.as<uint32_t>() + words - 1, 4, cudaMemcpyDeviceToHost, ctx_.compute));
      PSG_CUDA(cudaStreamSynchronize(ctx_.compute));
      ng = static_cast<uint64_t>(tail[0]) + tail[1];
    }
    rows = DevBuf(ctx_.pool, std::max<uint64_t>(ng, 1) * nc * 8, ctx_.compute);
    if (ng)
      launch_agg_emit_dense(aggt_, agg_cap_, cnt[1], bitmap.as<unsigned long long>(), prefix.as<uint32_t>(), nc,
                            kind.data(), idx.data(), rows.as<uint64_t>(), ctx_.compute);
  } else if (ng) {
    if (!known) {  // sparse fallback needs the exact count and range
      PSG_CUDA(cudaMemcpyAsync(counter.p, init, 24, cudaMemcpyHostToDevice, ctx_.compute));
      launch_agg_range(aggt_, agg_cap_, counter.as<unsigned long long>(), ctx_.compute);
      PSG_CUDA(cudaMemcpyAsync(cnt, counter.p, 24, cudaMemcpyDeviceToHost, ctx_.compute));
      PSG_CUDA(cudaStreamSynchronize(ctx_.compute));
      ng = cnt[0];
    }
    rows = DevBuf(ctx_.pool, std::max<uint64_t>(ng, 1) * nc * 8, ctx_.compute);
    DevBuf keys(ctx_.pool, nslots * 8, ctx_.compute), slots(ctx_.pool, nslots * 8, ctx_.compute);
    PSG_CUDA(cudaMemcpyAsync(counter.p, init, 24, cudaMemcpyHostToDevice, ctx_.compute));
    launch_agg_compact(aggt_, agg_cap_, keys.as<uint64_t>(), slots.as<unsigned long long>(),
                       counter.as<unsigned long long>(), ctx_.compute);
    // radix-sort only the key bits that vary: every key lies in [min, max] and shares their prefix
    int end_bit = 1;
    if (ng > 1 && cnt[1] != cnt[2]) end_bit = 64 - __builtin_clzll(cnt[1] ^ cnt[2]);
    DevBuf k2(ctx_.pool, ng * 8, ctx_.compute), s2(ctx_.pool, ng * 8, ctx_.compute);
    size_t tb = sort_pairs_i64(nullptr, nullptr, nullptr, nullptr, ng, end_bit, nullptr, 0, ctx_.compute);
    DevBuf tmp(ctx_.pool, std::max<size_t>(tb, 8), ctx_.compute);
    sort_pairs_i64(keys.as<uint64_t>(), k2.as<uint64_t>(), slots.as<unsigned long long>(), s2.as<unsigned long long>(), ng,
                   end_bit, tmp.p, tb, ctx_.compute);
    launch_agg_emit(aggt_, k2.as<uint64_t>(), s2.as<unsigned long long>(), ng, nc, kind.data(), idx.data(),
                    rows.as<uint64_t>(), ctx_.compute);
  }
  out.nrows = ng;
  if (want_rows) {
    uint64_t* dst = out.mutable_rows(ng * nc);
    if (ng) PSG_CUDA(cudaMemcpyAsync(dst, rows.p, ng * nc * 8, cudaMemcpyDeviceToHost, ctx_.compute));
    st_.result_bytes += ng * nc * 8;
  }
  PSG_CUDA(cudaStreamSynchronize(ctx_.compute));
}

void Execution::finalize_global(ResultRows& out) {
  const int nps = static_cast<int>(probe_sum_wire.size()), nbs = static_cast<int>(build_sum_wire.size());
  std::vector<uint64_t> acc(1 + nps + nbs);
  PSG_CUDA(cudaMemcpyAsync(acc.data(), global_acc_.p, acc.size() * 8, cudaMemcpyDeviceToHost, ctx_.compute));
  PSG_CUDA(cudaStreamSynchronize(ctx_.compute));
  st_.result_bytes += acc.size() * 8;
  if (acc[0] == 0) {
    out.nrows = 0;
    return;
  }
  out.nrows = 1;
  out.words.push_back(acc[0]);
  for (auto [side, k] : sum_order) out.words.push_back(side == 1 ? acc[1 + k] : acc[1 + nps + k]);
}

// ---------------------------------------------------------------------------------- run
/// Scope of a plan memory budget on the device pool: cleared on every exit path (a failed
/// budgeted query must not leave its budget on the context for the next one).
struct BudgetScope {
  DevicePool& pool;
  bool on;
  BudgetScope(DevicePool& p, uint64_t budget) : pool(p), on(budget != 0) {
    if (on) pool.set_budget(pool.used() + budget);
  }
  ~BudgetScope() {
    if (on) pool.set_budget(0);
  }
};

ResultRows Execution::run(bool want_rows) {
  const auto t0 = Clock::now();
  launches0_ = kernel_launch_count();
  jit0_ = jit_stats().compiles;
  ctx_.pool.reset_peak();
  BudgetScope budget_scope(ctx_.pool, plan_.memory_budget_bytes);
  PSG_TRACE_MSG("run: compile");
  cudaEvent_t ev0, ev1;
  PSG_CUDA(cudaEventCreate(&ev0));
  PSG_CUDA(cudaEventCreate(&ev1));
  PSG_CUDA(cudaEventRecord(ev0, ctx_.compute));
  std::unique_ptr<Timeline> timeline;
  if (Timeline::enabled()) {
    timeline = std::make_unique<Timeline>(ctx_.compute);
    ctx_.timeline = timeline.get();
  }
  struct TimelineScope {
    Ctx& c;
    ~TimelineScope() { c.timeline = nullptr; }
  } tl_scope{ctx_};
  compile();
  PSG_TRACE_MSG("run: compiled, build wire %zu cols, probe wire %zu cols", bsrc_.wire.size(), psrc_.wire.size());
  ResultRows out;
  out.schema = result_schema_;
  const int nr = ctx_.nranks;
  const int bkey = static_cast<int>(bsrc_.wire.require(shuffle_->build_key));
  const int pkey = static_cast<int>(psrc_.wire.require(shuffle_->probe_key));

  // Needed wire columns per side (projection pushdown past the shuffle).
  std::vector<int> bneed{bkey}, pneed{pkey};
  if (agg_) {
    for (int w : build_sum_wire) bneed.push_back(w);
    for (int w : probe_sum_wire) pneed.push_back(w);
  } else {
    for (size_t i = 0; i < bsrc_.wire.size(); ++i)
      if (static_cast<int>(i) != bkey) bneed.push_back(static_cast<int>(i));
    for (size_t i = 0; i < psrc_.wire.size(); ++i)
      if (static_cast<int>(i) != pkey) pneed.push_back(static_cast<int>(i));
  }
  // the build side's key is a late column: only rows passing the predicate and the local joins
  // need it (Q3 orders: 9% - most of its sectors are never read); the probe side's key is early
  // (its screen / table lookup needs it for every row that passes the predicate)
  RegMap bm = analyse(bsrc_, bneed, -1, true);
  RegMap pm = analyse(psrc_, pneed, pkey, true);
  for (size_t j = 0; j < bsrc_.chain.size(); ++j) bsrc_.chain[j].needed_payload = bm.payload_cols[j];
  for (size_t j = 0; j < psrc_.chain.size(); ++j) psrc_.chain[j].needed_payload = pm.payload_cols[j];

  if (!staged_) {
    // hash-table reservation for the ring regulation: the plan's estimate, else the reference
    // planner's fallback of a quarter of the budget (pipeline.cpp:588-593)
    uint64_t ht_reserve = plan_.ht_estimate_bytes;
    if (ht_reserve == 0 && plan_.memory_budget_bytes) ht_reserve = plan_.memory_budget_bytes / 4;
    session_ = std::make_unique<StreamSession>(ctx_, scan_list(bm, pm), plan_.memory_budget_bytes, ht_reserve);
  }
  const auto t_storage = Clock::now();
  PhaseTimer pt;
  pt.mark("compile", ctx_.compute);
  build_local_tables();
  pt.mark("local tables", ctx_.compute);
  const bool bdup = dup_chain(bsrc_), pdup = dup_chain(psrc_);  // expanding local joins

  // ---------------- build side ----------------
  ScanProgram bp = base_program(bsrc_, bm, true);
  std::vector<int> b_out;  // materialised columns: key first, then the rest of bneed
  for (int w : bneed) b_out.push_back(bm.reg_of.at(bsrc_.stage_refs.back()[w]));
  auto bfeed = open_feed(*bsrc_.scan, file_cols_of(bsrc_, bm));
  std::vector<Received> brecv;
  DevCols bmat;
  // Fused NVLink path (grouped aggregates, N > 1): no shuffle of rows at all — build keys are
  // inserted into, and probe rows aggregated in, the owner rank's table through peer memory.
  const bool p2p = nr > 1 && agg_ && grouped_ && ctx_.p2p && ctx_.symm_bytes > 0 && jit_available() && !bdup && !pdup;
  ctx_.symm_top = 0;
  DevBuf owner_hist;
  // Key-bitmap build: a grouped aggregate over a rank-indexed table whose build side carries
  // nothing but unique keys (Q3's orders) needs only the SET of build keys. The build scan then
  // sets each surviving key's bit in a bitmap over the zone-map key range (SINK_KEYBITS) - no
  // build rows are materialised, and at N > 1 none are shuffled: a SUM all-reduce of the rank
  // bitmaps (disjoint when the keys are unique; checked) is the global key set, the semi-join
  // screen of the probe side, and each rank keeps the bits it owns (partition_of) as its table.
  // Every decision below comes from all-reduced values, so all ranks agree. PSG_KEYBITS=0: off.
  bool kb_direct = false;
  long long kb_lo = 0;
  uint64_t kb_range = 0;
  DevBuf kb_cnt;  // [rows that set a bit (u64), flag (u32)]
  // peer-slab shuffle inputs, from the same all-reduce (N > 1): the probe columns' zone ranges
  // (bit-packed rows) and the largest probe side (slab capacity)
  std::vector<int64_t> slab_plo, slab_phi;
  uint64_t slab_max_rows = 0, probe_rows_all = 0;
  if (keybits_env() && agg_ && grouped_ && !p2p && !bdup && !ctx_.no_keybits && jit_available() && rank_table_env() &&
      kbits_mode() >= 1 && b_out.size() == 1 && build_sum_wire.empty() && ctx_.semijoin) {
    const ColRef kref = bsrc_.stage_refs.back()[bkey];
    if (kref.join < 0) {
      const size_t np = pneed.size();
      // MAX-reduced: [~lo, hi, probe rows, ~plo[k], phi[k]...]; SUM-reduced: [build rows, probe rows]
      std::vector<long long> mx(3 + 2 * np), sm(2, 0);
      long long lo = LLONG_MAX, hi = LLONG_MIN;
      zone_range(bsrc_.scan->paths, bsrc_.proj.file_idx[kref.idx], lo, hi);
      for (const auto& path : bsrc_.scan->paths) sm[0] += static_cast<long long>(ctx_.footers.get(path)->total_rows());
      for (const auto& path : psrc_.scan->paths) sm[1] += static_cast<long long>(ctx_.footers.get(path)->total_rows());
      mx[0] = ~lo, mx[1] = hi, mx[2] = sm[1];
      for (size_t k = 0; k < np; ++k) {
        long long a = LLONG_MAX, b = LLONG_MIN;
        const ColRef ref = psrc_.stage_refs.back()[pneed[k]];
        if (ref.join >= 0 || psrc_.wire.fields[pneed[k]].type != LType::Int64)
          a = LLONG_MIN, b = LLONG_MAX;  // not bounded by the zone maps: never packs
        else
          zone_range(psrc_.scan->paths, psrc_.proj.file_idx[ref.idx], a, b);
        mx[3 + k] = ~a, mx[3 + np + k] = b;
      }
      if (nr > 1) {  // one all-gather of every rank's vector; MAX / SUM reduced on the host
        const size_t nv = mx.size() + sm.size();
        std::vector<long long> mine(mx);
        mine.insert(mine.end(), sm.begin(), sm.end());
        DevBuf in(ctx_.pool, nv * 8, ctx_.compute), all(ctx_.pool, nv * 8 * nr, ctx_.compute);
        PSG_CUDA(cudaMemcpyAsync(in.p, mine.data(), nv * 8, cudaMemcpyHostToDevice, ctx_.compute));
        PSG_NCCL(ncclAllGather(in.p, all.p, nv, ncclInt64, ctx_.nccl, ctx_.compute));
        std::vector<long long> got(nv * nr);
        PSG_CUDA(cudaMemcpyAsync(got.data(), all.p, got.size() * 8, cudaMemcpyDeviceToHost, ctx_.compute));
        PSG_CUDA(cudaStreamSynchronize(ctx_.compute));
        for (size_t k = 0; k < mx.size(); ++k) {
          mx[k] = got[k];
          for (int r = 1; r < nr; ++r) mx[k] = std::max(mx[k], got[r * nv + k]);
        }
        for (size_t k = 0; k < sm.size(); ++k) {
          sm[k] = 0;
          for (int r = 0; r < nr; ++r) sm[k] += got[r * nv + mx.size() + k];
        }
      }
      lo = ~mx[0], hi = mx[1];
      slab_max_rows = static_cast<uint64_t>(mx[2]);
      probe_rows_all = static_cast<uint64_t>(sm[1]);
      for (size_t k = 0; k < np; ++k) slab_plo.push_back(~mx[3 + k]), slab_phi.push_back(mx[3 + np + k]);
      const uint64_t rows = static_cast<uint64_t>(sm[0]);
      const uint64_t range = hi >= lo ? static_cast<uint64_t>(hi) - static_cast<uint64_t>(lo) + 1 : 0;
      // the same tests as the materialising path, on the footer row count: a table big enough to
      // want a screen (one GPU), and a bitmap no larger than the Bloom filter it replaces
      const uint64_t cap = pow2_at_least(std::max<uint64_t>(2 * rows, 16));
      const int hw_est = 2 + static_cast<int>(probe_sum_wire.size()) <= 4 ? 4 : 8;
      const uint64_t bloom = std::min<uint64_t>(pow2_at_least(std::max<uint64_t>(rows / 2, 1024)), 8ull << 20);
      const bool screen = nr > 1 || (cap + 1) * hw_est * 8 > screen_min_bytes();
      if (screen && range != 0 && range <= (1ULL << 36) && lo != LLONG_MIN && range / 32 <= bloom * static_cast<uint64_t>(nr) &&
          (range + 63) / 64 < (1ULL << 32)) {
        kb_direct = true;
        kb_lo = lo;
        kb_range = range;
      }
    }
  }
  // N > 1: the local key bitmaps (and their duplicate flags) go into the symmetric heap, so every
  // rank ORs them through NVLink (k_or_own) instead of a SUM all-reduce; the heap also holds the
  // peer-slab outboxes when that path applies. One collective sizing (every input all-reduced).
  bool kb_heap = false;
  size_t kb_bits_off = 0, kb_cnt_off = 0;
  bool slab_possible = false;
  PackLayout slab_layout;
  uint64_t slab_cap = 0;
  if (kb_direct && nr > 1) {
    const uint64_t words64 = (kb_range + 63) / 64;
    if (!pdup && slab_env() && !ctx_.no_buckets && nr <= kMaxSlabPeers && pneed.size() >= 2 && pneed.size() <= 4 &&
        slab_plo.size() == pneed.size()) {
      slab_layout = plan_pack(slab_plo.data(), slab_phi.data(), static_cast<int>(pneed.size()));
      // every row, plus one partly filled chunk per (warp, destination) of the probe kernel
      slab_cap = std::max<uint64_t>(slab_max_rows, 1) + kSlabChunkSlack;
      const size_t sneed = 512 + static_cast<size_t>(nr) * slab_cap * 8;
      const bool budget_ok = plan_.memory_budget_bytes == 0 || sneed <= plan_.memory_budget_bytes / 2;
      // (packed rows of at most 63 bits: bit 63 marks the padding of partly filled chunks)
      slab_possible = slab_layout.fits && slab_layout.bits < 64 && budget_ok;
    }
    // PSG_KB_OR=0|1 forces the SUM all-reduce / the NVLink OR; default: the OR up to 4 ranks
    // (measured at N=2: key-bitmap phase 0.16 -> 0.10 ms; every rank reads all N bitmaps, so past 4
    // ranks NCCL's reduce-scatter + all-gather moves fewer bytes)
    static const int or_knob = [] {
      const char* e = std::getenv("PSG_KB_OR");
      return e ? std::atoi(e) : -1;
    }();
    const bool or_env = or_knob >= 0 ? or_knob != 0 : nr <= 4;
    const size_t bneed = ((words64 * 8 + 255) & ~size_t(255)) + 256;
    const size_t need = (or_env ? bneed : 0) + (slab_possible ? 512 + static_cast<size_t>(nr) * slab_cap * 8 + 256 : 0);
    if (need && ensure_symmetric(need)) {
      ctx_.symm_top = 0;
      if (or_env) {
        kb_bits_off = static_cast<size_t>(ctx_.symm_alloc(words64 * 8) - ctx_.symm);
        kb_cnt_off = static_cast<size_t>(ctx_.symm_alloc(16) - ctx_.symm);
        kb_heap = true;
      }
    } else {
      slab_possible = false;
    }
  }
  if (kb_direct) {
    const uint64_t words64 = (kb_range + 63) / 64;
    uint32_t* kbits = nullptr;
    unsigned long long* kcnt = nullptr;
    if (kb_heap) {
      kbits = reinterpret_cast<uint32_t*>(ctx_.symm + kb_bits_off);
      kcnt = reinterpret_cast<unsigned long long*>(ctx_.symm + kb_cnt_off);
    } else {
      agg_kbits_ = DevBuf(ctx_.pool, words64 * 8, ctx_.compute);
      kb_cnt = DevBuf(ctx_.pool, 16, ctx_.compute);
      kbits = agg_kbits_.as<uint32_t>();
      kcnt = kb_cnt.as<unsigned long long>();
    }
    PSG_CUDA(cudaMemsetAsync(kbits, 0, words64 * 8, ctx_.compute));
    PSG_CUDA(cudaMemsetAsync(kcnt, 0, 16, ctx_.compute));
    ScanProgram p = bp;
    p.sink = SINK_KEYBITS;
    p.staged_ok = 1;  // PSTO batches / staged images: 16-byte aligned chunks with tail padding
    p.key_reg = b_out[0];
    p.kb_bits = kbits;
    p.kb_min = kb_lo;
    p.kb_range = kb_range;
    p.kb_count = kcnt;
    p.kb_flag = nullptr;  // bits by reductions; duplicates = fewer set bits than rows (checked below)
    BatchView v;
    while (bfeed->next(v)) {
      run_scan(p, v, false);
      bfeed->done();
      st_.ingest_bytes += v.bytes;
    }
  } else if (nr == 1 || p2p) {
    bmat = alloc_cols(b_out.size(), std::max<uint64_t>(bfeed->total_rows, 1));
    if (p2p) {
      owner_hist = DevBuf(ctx_.pool, nr * 8, ctx_.compute);
      PSG_CUDA(cudaMemsetAsync(owner_hist.p, 0, nr * 8, ctx_.compute));
    }
    BatchView v;
    std::vector<DevCols> parts;
    while (bfeed->next(v)) {
      if (bdup)
        parts.push_back(materialize_chain(bsrc_, bm, v, b_out));
      else
        materialize_into(bmat, bp, v, b_out, p2p ? b_out[0] : -1, p2p ? &owner_hist : nullptr, false, true);
      bfeed->done();
      st_.ingest_bytes += v.bytes;
    }
    if (bdup)
      bmat = concat_cols(parts, b_out.size());
    else
      read_count(bmat);
  } else {
    // agree on the wave count (the reference's kDoneFlag vote, pipeline.cpp:696-722)
    uint64_t waves = bfeed->nbatches;
    DevBuf wv(ctx_.pool, 8, ctx_.compute);
    PSG_CUDA(cudaMemcpyAsync(wv.p, &waves, 8, cudaMemcpyHostToDevice, ctx_.compute));
    PSG_NCCL(ncclAllReduce(wv.p, wv.p, 1, ncclUint64, ncclMax, ctx_.nccl, ctx_.compute));
    PSG_CUDA(cudaMemcpyAsync(&waves, wv.p, 8, cudaMemcpyDeviceToHost, ctx_.compute));
    PSG_CUDA(cudaStreamSynchronize(ctx_.compute));
    for (uint64_t w = 0; w < waves; ++w) {
      BatchView v;
      const bool have = bfeed->next(v);
      DevCols mat = alloc_cols(b_out.size(), std::max<uint64_t>(have ? v.rows : 1, 1));
      DevBuf pc(ctx_.pool, nr * 8, ctx_.compute);
      PSG_CUDA(cudaMemsetAsync(pc.p, 0, nr * 8, ctx_.compute));
      if (have && bdup) {
        mat = materialize_chain(bsrc_, bm, v, b_out);
        launch_part_hist(mat.cols[0].as<uint64_t>(), mat.rows, nr, pc.as<unsigned long long>(), ctx_.compute);
        bfeed->done();
        st_.ingest_bytes += v.bytes;
      } else if (have) {
        materialize_into(mat, bp, v, b_out, b_out[0], &pc, false, true);
        bfeed->done();
        st_.ingest_bytes += v.bytes;
      }
      brecv.push_back(exchange(mat, static_cast<int>(b_out.size()), 0, pc, have));
    }
  }
  pt.mark("build side scan", ctx_.compute);
  uint64_t build_rows = 0;
  uint64_t p2p_max_rows = 0;
  if (p2p) {
    // rows each owner will hold = sum over ranks of the per-owner histograms
    std::vector<uint64_t> local(nr), owners(nr);
    PSG_CUDA(cudaMemcpyAsync(local.data(), owner_hist.p, nr * 8, cudaMemcpyDeviceToHost, ctx_.compute));
    PSG_NCCL(ncclAllReduce(owner_hist.p, owner_hist.p, nr, ncclUint64, ncclSum, ctx_.nccl, ctx_.compute));
    PSG_CUDA(cudaMemcpyAsync(owners.data(), owner_hist.p, nr * 8, cudaMemcpyDeviceToHost, ctx_.compute));
    PSG_CUDA(cudaStreamSynchronize(ctx_.compute));
    build_rows = owners[ctx_.rank];
    for (uint64_t x : owners) p2p_max_rows = std::max(p2p_max_rows, x);
    st_.bytes_received += (owners[ctx_.rank] - local[ctx_.rank]) * 8 * b_out.size();
  } else if (nr == 1) {
    build_rows = bmat.rows;
  } else {
    for (auto& r : brecv) build_rows += r.rows;
  }

  // Program over materialised build rows: reg k = column k of the materialised batch.
  auto batch_program = [&](int ncols) {
    ScanProgram p;
    std::memset(&p, 0, sizeof p);
    p.n_in = ncols;
    p.n_pred = 0;
    p.n_early = std::min(1, ncols);
    p.n_regs = std::max(1, ncols);
    p.part_key_reg = -1;
    p.key_reg = 0;
    return p;
  };
  std::vector<Segment> bsegs;
  if (kb_direct) {
    // (no build rows: the key bitmap is the whole build side)
  } else if (nr == 1 || p2p) {
    Segment sg;
    std::memset(&sg, 0, sizeof sg);
    for (size_t c = 0; c < b_out.size(); ++c) sg.col[c] = bmat.cols[c].as<uint64_t>();
    sg.rows = bmat.rows;
    if (sg.rows) bsegs.push_back(sg);
  } else {
    for (auto& r : brecv)
      for (auto& s : r.segs) bsegs.push_back(s);
  }
  DevBuf bseg_holder;
  BatchView bview = upload_segments(bsegs, bseg_holder);

  // For no-aggregate plans the build side becomes a CSR table of full wire rows.
  std::unique_ptr<LocalTable> final_table;
  // Bloom filter over the build keys: at one GPU it screens probes when the hot table would not
  // stay L2-resident; at N GPUs every rank's filter is all-gathered so the probe side can drop
  // rows whose key is absent on its owner before the shuffle (semi-join reduction). All ranks
  // size the filter from the largest build side so the filters line up.
  DevBuf semi_all;
  uint64_t bloom_words = 0;
  const bool semi = agg_ && nr > 1 && ctx_.semijoin && !p2p;
  if (agg_ && !kb_direct) {
    uint64_t sized_rows = build_rows;
    if (semi) {
      DevBuf mv(ctx_.pool, 8, ctx_.compute);
      PSG_CUDA(cudaMemcpyAsync(mv.p, &sized_rows, 8, cudaMemcpyHostToDevice, ctx_.compute));
      PSG_NCCL(ncclAllReduce(mv.p, mv.p, 1, ncclUint64, ncclMax, ctx_.nccl, ctx_.compute));
      PSG_CUDA(cudaMemcpyAsync(&sized_rows, mv.p, 8, cudaMemcpyDeviceToHost, ctx_.compute));
      PSG_CUDA(cudaStreamSynchronize(ctx_.compute));
    }
    const uint64_t cap = pow2_at_least(std::max<uint64_t>(2 * build_rows, 16));
    const int hw_est = 2 + static_cast<int>(probe_sum_wire.size()) <= 4 ? 4 : 8;
    // a one-GPU table larger than ~L2/2.5 gets a membership screen (screen_min_bytes)
    if (semi || ((cap + 1) * hw_est * 8 > screen_min_bytes() && ctx_.semijoin))
      bloom_words = std::min<uint64_t>(pow2_at_least(std::max<uint64_t>(sized_rows / 2, 1024)), 8ull << 20);
  }
  DevBuf peers_dev;
  bool p2p_ok = p2p;
  if (p2p) {
    // symmetric tables: identical capacity on every rank (sized from the largest owner), carved
    // from the IPC-mapped heap in the same order everywhere so peers find them at equal offsets
    p2p_ok = build_symmetric_agg_table(p2p_max_rows, ctx_.semijoin);
    st_.agg_table = 5;
    if (!p2p_ok) throw Error(PSG_ERR_MEMORY_EXCEEDED, "symmetric heap too small for the aggregation table (raise PSG_SYMM_MB)");
    std::vector<AggPeer> peers(nr);
    const size_t hot_off = reinterpret_cast<uint8_t*>(aggt_.hot) - ctx_.symm;
    const size_t cold_off = reinterpret_cast<uint8_t*>(aggt_.cold) - ctx_.symm;
    const size_t bloom_off = aggt_.bloom ? reinterpret_cast<uint8_t*>(aggt_.bloom) - ctx_.symm : 0;
    for (int q = 0; q < nr; ++q) {
      peers[q].hot = reinterpret_cast<uint64_t*>(ctx_.symm_peer[q] + hot_off);
      peers[q].cold = reinterpret_cast<uint64_t*>(ctx_.symm_peer[q] + cold_off);
      peers[q].bloom = aggt_.bloom ? reinterpret_cast<uint32_t*>(ctx_.symm_peer[q] + bloom_off) : nullptr;
      peers[q].pad = 0;
    }
    peers_dev = DevBuf(ctx_.pool, nr * sizeof(AggPeer), ctx_.compute);
    PSG_CUDA(cudaMemcpyAsync(peers_dev.p, peers.data(), nr * sizeof(AggPeer), cudaMemcpyHostToDevice, ctx_.compute));
    gpu_barrier();  // every owner's table is initialised before anyone inserts
    ScanProgram p = batch_program(static_cast<int>(b_out.size()));
    p.sink = SINK_BUILD;
    p.agg = aggt_;
    p.remote = 1;
    p.peers = peers_dev.as<AggPeer>();
    p.nparts = nr;
    p.n_sum = static_cast<int>(build_sum_wire.size());
    for (int b = 0; b < p.n_sum; ++b) p.sum_reg[b] = 1 + b;
    run_scan(p, bview, false);
    gpu_barrier();  // all inserts (and Bloom bits) landed in every owner's table
    if (aggt_.bloom) {
      bloom_words = aggt_.bloom_mask + 1;
      semi_all = DevBuf(ctx_.pool, static_cast<size_t>(nr) * bloom_words * 4, ctx_.compute);
      for (int q = 0; q < nr; ++q)
        PSG_CUDA(cudaMemcpyAsync(semi_all.as<uint32_t>() + q * bloom_words, peers[q].bloom, bloom_words * 4,
                                 cudaMemcpyDeviceToDevice, ctx_.compute));
    }
  } else if (agg_) {
    pt.mark("  pre agg alloc", ctx_.compute);
    // Dense build keys at one GPU: an exact membership bitmap replaces the Bloom filter (no false
    // positives, 1 bit per key of the range; o_orderkey at SF100: 19 MB vs 32 MB). At N > 1 every
    // rank sets its own bitmap over the ALL-REDUCED key range from the build keys it owns; the OR
    // of the rank bitmaps (a SUM all-reduce: owners are disjoint) is the exact semi-join screen of
    // the probe side, and a rank's own bitmap indexes its rank-indexed table.
    const bool kbits_env = kbits_mode() >= 1;
    // Rank-indexed table (grouped, unique dense build keys): the key bitmap is set from the build
    // keys first (with a duplicate check) and its 64-bit words' popcount prefix turns a key into
    // its rank = its slot; the table is then exactly one slot per build key in key order, written
    // by plain stores. PSG_RANK_TABLE=0: the hashed table.
    const bool rank_env = rank_table_env();
    long long krange_lo = 0;
    uint64_t krange = 0;
    const bool rank_ok = grouped_ && rank_env && jit_available() && !p2p;
    auto rank_records = [&](uint64_t kwords64) {  // popcount prefix per 64-bit word + interleaved {bits, rank} records
      agg_krank_ = DevBuf(ctx_.pool, kwords64 * 4, ctx_.compute);
      static const bool fused = [] {  // PSG_RANK_FUSED=0: popc64 + CUB scan + krec build (measurement knob)
        const char* e = std::getenv("PSG_RANK_FUSED");
        return !(e && std::string(e) == "0");
      }();
      if (fused && rank_tiles(kwords64) <= 16384) {  // (each tile sums the earlier tiles' counts)
        DevBuf ts(ctx_.pool, rank_tiles(kwords64) * 4, ctx_.compute);
        agg_krec_ = DevBuf(ctx_.pool, kwords64 * 16, ctx_.compute);
        launch_rank_records(agg_kbits_.as<unsigned long long>(), kwords64, ts.as<uint32_t>(), agg_krank_.as<uint32_t>(),
                            agg_krec_.as<unsigned long long>(), ctx_.compute);
        return;
      }
      DevBuf cnt(ctx_.pool, kwords64 * 4, ctx_.compute);
      launch_popc64(agg_kbits_.as<unsigned long long>(), kwords64, cnt.as<uint32_t>(), ctx_.compute);
      const size_t tb = exclusive_scan_u32(nullptr, nullptr, kwords64, nullptr, 0, ctx_.compute);
      DevBuf tmp(ctx_.pool, tb, ctx_.compute);
      exclusive_scan_u32(cnt.as<uint32_t>(), agg_krank_.as<uint32_t>(), kwords64, tmp.p, tb, ctx_.compute);
      agg_krec_ = DevBuf(ctx_.pool, kwords64 * 16, ctx_.compute);
      launch_krec_build(agg_kbits_.as<unsigned long long>(), agg_krank_.as<uint32_t>(), kwords64,
                        agg_krec_.as<unsigned long long>(), ctx_.compute);
    };
    if (kb_direct) {
      // the key bitmap was set by the build scan itself: N > 1 all-reduces it into the global key
      // set (semi_all) and keeps the bits this rank owns; one host read checks the key counts
      const uint64_t words64 = (kb_range + 63) / 64;
      DevBuf cnts(ctx_.pool, 32, ctx_.compute);  // [own bits, global bits, overlap, summed rows]
      PSG_CUDA(cudaMemsetAsync(cnts.p, 0, 32, ctx_.compute));
      if (nr > 1 && kb_heap) {
        // the owned-bit masks of one period of words (power-of-two N): computed before the barrier,
        // so off the critical path; PSG_OWN_TABLE=0: partition_of per set bit inside k_or_own
        static const bool own_table_env = [] {
          const char* e = std::getenv("PSG_OWN_TABLE");
          return !(e && e[0] == '0');
        }();
        const uint32_t period = own_table_env ? own_period(nr) : 0;
        DevBuf own_tbl;
        if (period) {
          own_tbl = DevBuf(ctx_.pool, static_cast<size_t>(period) * 8, ctx_.compute);
          launch_own_table(kb_lo, nr, ctx_.rank, own_tbl.as<unsigned long long>(), ctx_.compute);
        }
        gpu_barrier();  // every rank's local bitmap and flag are complete
        pt.mark("  barrier (rank bitmaps)", ctx_.compute);
        semi_all = DevBuf(ctx_.pool, (words64 + 1) * 8, ctx_.compute);
        agg_kbits_ = DevBuf(ctx_.pool, words64 * 8, ctx_.compute);
        OrPeers op{};
        op.n = nr;
        for (int r = 0; r < nr; ++r) {
          op.bits[r] = reinterpret_cast<const unsigned long long*>(ctx_.symm_peer[r] + kb_bits_off);
          op.rows[r] = reinterpret_cast<const unsigned long long*>(ctx_.symm_peer[r] + kb_cnt_off);
        }
        launch_or_own(op, words64, kb_lo, ctx_.rank, semi_all.as<unsigned long long>(), agg_kbits_.as<unsigned long long>(),
                      cnts.as<unsigned long long>(), ctx_.compute, period ? own_tbl.as<unsigned long long>() : nullptr,
                      period);
        pt.mark("  NVLink OR of the rank bitmaps", ctx_.compute);
        // (a peer may still read this rank's local bitmap: it is rewritten only by the next query's
        // build scan, which follows this query's collectives)
      } else if (nr > 1) {
        // (+1 word: the probe reads the global bitmap in aligned 16-byte chunks)
        semi_all = DevBuf(ctx_.pool, (words64 + 1) * 8, ctx_.compute);
        PSG_NCCL(ncclAllReduce(agg_kbits_.p, semi_all.p, words64, ncclUint64, ncclSum, ctx_.nccl, ctx_.compute));
        PSG_NCCL(ncclAllReduce(kb_cnt.p, kb_cnt.p, 1, ncclUint64, ncclSum, ctx_.nccl, ctx_.compute));
        PSG_NCCL(ncclAllReduce(kb_cnt.as<unsigned long long>() + 1, kb_cnt.as<unsigned long long>() + 1, 1, ncclUint64,
                               ncclMax, ctx_.nccl, ctx_.compute));
        launch_own_mask(semi_all.as<unsigned long long>(), agg_kbits_.as<unsigned long long>(), words64, kb_lo, nr,
                        ctx_.rank, cnts.as<unsigned long long>(), ctx_.compute);
      }
      // the rank records of the (own) bitmap are queued before the host read: at one GPU its
      // popcount (last prefix + last word) is the duplicate check
      rank_records((kb_range + 63) / 64);
      const uint64_t wl = (kb_range + 63) / 64 - 1;
      const auto* kc = kb_cnt.p ? kb_cnt.as<unsigned long long>() : reinterpret_cast<const unsigned long long*>(ctx_.symm + kb_cnt_off);
      const auto* cw = cnts.as<unsigned long long>();
      uint64_t h[8];
      read_words({{kc, false}, {kc + 1, false}, {cw, false}, {cw + 1, false}, {cw + 2, false}, {cw + 3, false},
                  {agg_krank_.as<uint32_t>() + wl, true}, {agg_kbits_.as<unsigned long long>() + wl, false}},
                 h);
      const uint32_t last_rank = static_cast<uint32_t>(h[6]);
      const uint64_t last_word = h[7];
      pt.mark("  key bitmap (global, own bits)", ctx_.compute);
      const uint64_t rows_set = h[0];
      if (kb_heap) {
        // overlaps and the summed row counts of every rank: identical on all ranks
        if (h[4] != 0 || h[5] != h[3] || h[3] == 0 || h[3] >= (1ULL << 32)) throw KeybitsRetry();
        build_rows = h[2];
      } else if (nr > 1) {
        // (rows_set is the all-reduced sum) a repeated key left fewer bits than rows; across ranks
        // the SUM all-reduce carried: fewer global bits than rows as well
        if (rows_set == 0 || rows_set >= (1ULL << 32) || h[3] != rows_set) throw KeybitsRetry();
        build_rows = h[2];
      } else {
        const uint64_t bits_set = static_cast<uint64_t>(last_rank) + static_cast<uint64_t>(__builtin_popcountll(last_word));
        if (rows_set == 0 || rows_set >= (1ULL << 32) || bits_set != rows_set) throw KeybitsRetry();
        build_rows = rows_set;
      }
      krange_lo = kb_lo;
      krange = kb_range;
      bloom_words = 0;
    } else if (nr > 1 && semi && kbits_env && (rank_ok || kbits_mode() >= 2)) {
      DevBuf mm(ctx_.pool, 16, ctx_.compute);
      const long long init[2] = {LLONG_MAX, LLONG_MIN};
      PSG_CUDA(cudaMemcpyAsync(mm.p, init, 16, cudaMemcpyHostToDevice, ctx_.compute));
      for (const auto& sg : bsegs) launch_minmax_i64(sg.col[0], sg.rows, mm.as<long long>(), ctx_.compute);
      long long lohi[2];
      PSG_CUDA(cudaMemcpyAsync(lohi, mm.p, 16, cudaMemcpyDeviceToHost, ctx_.compute));
      PSG_CUDA(cudaStreamSynchronize(ctx_.compute));
      long long enc[2] = {~lohi[0], lohi[1]};  // max(~lo) = ~min(lo)
      PSG_CUDA(cudaMemcpyAsync(mm.p, enc, 16, cudaMemcpyHostToDevice, ctx_.compute));
      PSG_NCCL(ncclAllReduce(mm.p, mm.p, 2, ncclInt64, ncclMax, ctx_.nccl, ctx_.compute));
      PSG_CUDA(cudaMemcpyAsync(enc, mm.p, 16, cudaMemcpyDeviceToHost, ctx_.compute));
      PSG_CUDA(cudaStreamSynchronize(ctx_.compute));
      const long long lo = ~enc[0], hi = enc[1];
      const uint64_t range = hi >= lo ? static_cast<uint64_t>(hi) - static_cast<uint64_t>(lo) + 1 : 0;
      // every rank decides from all-reduced numbers only (same choice everywhere); a bitmap of
      // <= 32 x the largest Bloom filter (the Bloom would be ~16 bits per key)
      if (range != 0 && range <= (1ULL << 36) && range / 32 <= static_cast<uint64_t>(nr) * bloom_words) {
        krange_lo = lo;
        krange = range;
        bloom_words = 0;
      }
    } else if (nr == 1 && bloom_words && kbits_env && bmat.rows) {
      // the key range: from the build scan's footer zone maps when the key is one of its columns
      // (a superset of the surviving keys' range: no kernel, no host round trip), else measured
      long long lohi[2] = {LLONG_MAX, LLONG_MIN};
      const ColRef kref = bsrc_.stage_refs.back()[bkey];
      if (kref.join < 0) {
        zone_range(bsrc_.scan->paths, bsrc_.proj.file_idx[kref.idx], lohi[0], lohi[1]);
      } else {
        DevBuf mm(ctx_.pool, 16, ctx_.compute);
        PSG_CUDA(cudaMemcpyAsync(mm.p, lohi, 16, cudaMemcpyHostToDevice, ctx_.compute));
        launch_minmax_i64(bmat.cols[0].as<uint64_t>(), bmat.rows, mm.as<long long>(), ctx_.compute);
        PSG_CUDA(cudaMemcpyAsync(lohi, mm.p, 16, cudaMemcpyDeviceToHost, ctx_.compute));
        PSG_CUDA(cudaStreamSynchronize(ctx_.compute));
      }
      const uint64_t range = static_cast<uint64_t>(lohi[1]) - static_cast<uint64_t>(lohi[0]) + 1;
      if (range != 0 && range <= (1ULL << 36) && range / 32 <= bloom_words) {  // no larger than the Bloom
        krange_lo = lohi[0];
        krange = range;
        bloom_words = 0;
      }
    }
    bool rank_mode = false;
    const uint64_t kwords64 = (krange + 63) / 64;
    if (kb_direct) {
      rank_mode = true;  // (rank records queued with the key-bitmap check above)
    } else if (krange && rank_ok && krange_lo != LLONG_MIN && kwords64 < (1ULL << 32) && build_rows > 0 &&
               build_rows < (1ULL << 32)) {
      agg_kbits_ = DevBuf(ctx_.pool, kwords64 * 8, ctx_.compute);
      DevBuf dup(ctx_.pool, 4, ctx_.compute);
      PSG_CUDA(cudaMemsetAsync(agg_kbits_.p, 0, kwords64 * 8, ctx_.compute));
      PSG_CUDA(cudaMemsetAsync(dup.p, 0, 4, ctx_.compute));
      for (const auto& sg : bsegs)
        launch_bitmap_set(sg.col[0], sg.rows, krange_lo, agg_kbits_.as<uint32_t>(), dup.as<unsigned int>(), ctx_.compute);
      unsigned int d = 1;
      PSG_CUDA(cudaMemcpyAsync(&d, dup.p, 4, cudaMemcpyDeviceToHost, ctx_.compute));
      PSG_CUDA(cudaStreamSynchronize(ctx_.compute));
      pt.mark("  key bitmap + dup check", ctx_.compute);
      if (!d) {
        rank_records(kwords64);
        rank_mode = true;
      }
    }
    pt.mark("  rank records", ctx_.compute);
    // (a rank that owns no keys at N > 1 keeps a one-slot table nobody probes)
    build_agg_table(build_rows, bloom_words, rank_mode ? std::max<uint64_t>(build_rows, 1) : 0);
    st_.agg_table = rank_mode ? 4 : (krange ? 3 : (bloom_words ? 2 : 1));
    if (krange) {
      if (!rank_mode) {  // the insert below sets the bits
        const uint64_t words = (krange + 31) / 32;
        agg_kbits_ = DevBuf(ctx_.pool, words * 4, ctx_.compute);
        PSG_CUDA(cudaMemsetAsync(agg_kbits_.p, 0, words * 4, ctx_.compute));
      }
      aggt_.kbits = agg_kbits_.as<uint32_t>();
      aggt_.kmin = krange_lo;
      aggt_.krange = krange;
      if (rank_mode) {
        aggt_.krank = agg_krank_.as<uint32_t>();
        aggt_.krec = agg_krec_.as<unsigned long long>();
      }
    }
    pt.mark("  agg table", ctx_.compute);
    // one GPU, rank table, fused probe: bucketed aggregation (the hot table is then only the target
    // of bucket overflow - zeroed instead of initialised with keys)
    // Peer-slab shuffle (N > 1, key-bitmap build): probe rows owned by another rank travel as one
    // bit-packed word stored by the probe kernel straight into the owner's receive slab over
    // NVLink (symmetric heap, one region per source rank, sized for the largest probe side), the
    // owners fold them into their buckets after a device-side barrier. PSG_SLAB=0: NCCL shuffle.
    // (every input of these decisions is all-reduced or plan-wide: all ranks agree; the heap was
    // sized with the key bitmaps above)
    const bool slab_cand = slab_possible && ctx_.symm_bytes > 0;
    if (rank_mode && (nr == 1 || slab_cand) && grouped_ && !pdup)
      bucket_mode_ = slab_cand ? setup_buckets(slab_plo.data() + 1, slab_phi.data() + 1, probe_rows_all) : setup_buckets();
    if (slab_cand && bucket_mode_) {
      uint8_t* cnt = ctx_.symm_alloc(static_cast<size_t>(nr) * 8);
      uint8_t* slab = ctx_.symm_alloc(static_cast<size_t>(nr) * slab_cap * 8);
      if (!cnt || !slab) throw Error(PSG_ERR_INTERNAL, "symmetric heap layout");
      slab_mode_ = true;
      slab_pack_ = std::move(slab_layout);
      slab_cap_ = slab_cap;
      slab_cnt_off_ = static_cast<size_t>(cnt - ctx_.symm);
      slab_off_ = static_cast<size_t>(slab - ctx_.symm);
      slab_grec_ = DevBuf(ctx_.pool, kwords64 * 16, ctx_.compute);
      launch_krec_build(semi_all.as<unsigned long long>(), agg_krank_.as<uint32_t>(), kwords64,
                        slab_grec_.as<unsigned long long>(), ctx_.compute);
    } else if (nr > 1) {
      bucket_mode_ = false;  // the NCCL shuffle's consume kernel updates the table directly
    }
    // packed accumulators serve the hot table's atomics: not needed when buckets take every row
    // (a collective at N > 1; bucket_mode_ is the same on every rank)
    if (!bucket_mode_) pack_accumulators();
    pt.mark("  pack accumulators", ctx_.compute);
    pt.mark("  agg alloc+init", ctx_.compute);
    ScanProgram p = batch_program(static_cast<int>(b_out.size()));
    p.sink = SINK_BUILD;
    p.agg = aggt_;
    p.n_sum = static_cast<int>(build_sum_wire.size());
    for (int b = 0; b < p.n_sum; ++b) p.sum_reg[b] = 1 + b;
    // N > 1 with the Bloom screen: the filter is set from the received keys in a separate pass and
    // all-gathered first, then the table insert runs on the aux stream while the probe side scans,
    // semi-join-screens, partitions and shuffles on the compute stream; the compute stream joins
    // the insert only where the table is first used (consume, or the in-place owner probe).
    // PSG_BUILD_OVERLAP=0: off.
    static const bool overlap_env = [] {
      const char* e = std::getenv("PSG_BUILD_OVERLAP");
      return !(e && std::string(e) == "0");
    }();
    if (rank_mode) {
      // hot slots from the bitmap (slot order) once, cold slots (build sums) per build segment
      bool first = true;
      for (const auto& sg : bsegs) {
        RankSums rs{};
        for (int b = 0; b < p.n_sum; ++b) rs.col[b] = sg.col[1 + b];
        launch_rank_build(aggt_, sg.col[0], rs, sg.rows, first, !bucket_mode_, ctx_.compute);
        first = false;
      }
      if (first) launch_rank_build(aggt_, nullptr, RankSums{}, 0, true, !bucket_mode_, ctx_.compute);
    } else if (semi && !krange && aggt_.bloom && overlap_env) {
      for (const auto& sg : bsegs) launch_bloom_keys(sg.col[0], sg.rows, aggt_.bloom, aggt_.bloom_shift, ctx_.compute);
      PSG_CUDA(cudaEventRecord(build_fork_.get(), ctx_.compute));
      PSG_CUDA(cudaStreamWaitEvent(ctx_.comm, build_fork_.get(), 0));
      p.agg.bloom = nullptr;
      if (bview.nsegs) fused_scan(p, bview.d_segs, bview.d_tile_seg, bview.nsegs, bview.ntiles, ctx_.comm);
      PSG_CUDA(cudaEventRecord(build_done_.get(), ctx_.comm));
      build_pending_ = true;
      semi_all = DevBuf(ctx_.pool, static_cast<size_t>(nr) * bloom_words * 4, ctx_.compute);
      PSG_NCCL(ncclAllGather(agg_bloom_.p, semi_all.p, bloom_words * 4, ncclUint8, ctx_.nccl, ctx_.compute));
    } else {
      run_scan(p, bview, false);  // also sets the Bloom (or key-bitmap) bits of every inserted key
    }
    if (build_pending_) {
      // (the Bloom filters were all-gathered above)
    } else if (kb_direct) {
      // (semi_all is the all-reduced global key bitmap already)
    } else if (semi && krange) {  // disjoint bits: SUM == OR; out of place (the rank keeps its own)
      const uint64_t words = (krange + 31) / 32;
      semi_all = DevBuf(ctx_.pool, words * 4, ctx_.compute);
      PSG_NCCL(ncclAllReduce(agg_kbits_.p, semi_all.p, words, ncclUint32, ncclSum, ctx_.nccl, ctx_.compute));
    } else if (semi) {
      semi_all = DevBuf(ctx_.pool, static_cast<size_t>(nr) * bloom_words * 4, ctx_.compute);
      PSG_NCCL(ncclAllGather(agg_bloom_.p, semi_all.p, bloom_words * 4, ncclUint8, ctx_.nccl, ctx_.compute));
    }
    if (!grouped_) {
      global_acc_ = DevBuf(ctx_.pool, (2 * kMaxSums + 1) * 8, ctx_.compute);
      PSG_CUDA(cudaMemsetAsync(global_acc_.p, 0, (2 * kMaxSums + 1) * 8, ctx_.compute));
    }
  } else {
    // materialise received build rows contiguously, then CSR-build with payload = other columns
    const int nc = static_cast<int>(b_out.size());
    DevCols all = alloc_cols(nc, std::max<uint64_t>(build_rows, 1));
    ScanProgram p = batch_program(nc);
    p.n_early = nc;
    std::vector<int> regs(nc);
    std::iota(regs.begin(), regs.end(), 0);
    materialize_into(all, p, bview, regs, -1, nullptr);
    const uint64_t n = read_count(all);
    final_table = std::make_unique<LocalTable>();
    auto& t = *final_table;
    t.cap = pow2_at_least(std::max<uint64_t>(2 * n, 16));
    t.keys = DevBuf(ctx_.pool, t.cap * 8, ctx_.compute);
    t.cnt = DevBuf(ctx_.pool, (t.cap + 1) * 4, ctx_.compute);
    t.start = DevBuf(ctx_.pool, (t.cap + 1) * 4, ctx_.compute);
    DevBuf cursor(ctx_.pool, (t.cap + 1) * 4, ctx_.compute), maxc(ctx_.pool, 4, ctx_.compute);
    PSG_CUDA(cudaMemsetAsync(maxc.p, 0, 4, ctx_.compute));
    PSG_CUDA(cudaMemsetAsync(cursor.p, 0, (t.cap + 1) * 4, ctx_.compute));
    launch_local_init(t.keys.as<uint64_t>(), t.cnt.as<uint32_t>(), t.cap, ctx_.compute);
    launch_local_count(t.keys.as<uint64_t>(), t.cnt.as<uint32_t>(), t.cap - 1, shift_of(t.cap), all.cols[0].as<uint64_t>(), n,
                       maxc.as<unsigned>(), ctx_.compute);
    size_t tb = exclusive_scan_u32(nullptr, nullptr, t.cap + 1, nullptr, 0, ctx_.compute);
    DevBuf tmp(ctx_.pool, tb, ctx_.compute);
    exclusive_scan_u32(t.cnt.as<uint32_t>(), t.start.as<uint32_t>(), t.cap + 1, tmp.p, tb, ctx_.compute);
    std::vector<const uint64_t*> src;
    std::vector<uint64_t*> dst;
    for (int c = 1; c < nc; ++c) {
      t.payload.emplace_back(ctx_.pool, std::max<uint64_t>(n, 1) * 8, ctx_.compute);
      src.push_back(all.cols[c].as<uint64_t>());
      dst.push_back(t.payload.back().as<uint64_t>());
    }
    launch_local_fill(t.keys.as<uint64_t>(), t.start.as<uint32_t>(), cursor.as<uint32_t>(), t.cap - 1, shift_of(t.cap),
                      all.cols[0].as<uint64_t>(), src.data(), dst.data(), nc - 1, n, ctx_.compute);
    t.dev.keys = t.keys.as<uint64_t>();
    t.dev.cnt = t.cnt.as<uint32_t>();
    t.dev.start = t.start.as<uint32_t>();
    t.dev.mask = t.cap - 1;
    t.dev.shift = shift_of(t.cap);
    t.dev.npayload = nc - 1;
    for (int c = 0; c < nc - 1; ++c) t.dev.payload[c] = t.payload[c].as<uint64_t>();
    PSG_CUDA(cudaStreamSynchronize(ctx_.compute));
  }
  // the received build rows stay allocated until the (possibly concurrent) insert has finished
  std::vector<Received> brecv_hold;
  DevCols bmat_hold;
  if (build_pending_) {
    brecv_hold = std::move(brecv);
    bmat_hold = std::move(bmat);
  }
  brecv.clear();
  bmat = DevCols{};
  auto join_build = [&] {
    if (!build_pending_) return;
    PSG_CUDA(cudaStreamWaitEvent(ctx_.compute, build_done_.get(), 0));
    build_pending_ = false;
    brecv_hold.clear();
    bmat_hold = DevCols{};
  };

  pt.mark("build table", ctx_.compute);
  // ---------------- probe side ----------------
  ScanProgram pp = base_program(psrc_, pm, true);
  std::vector<int> p_out;
  for (int w : pneed) p_out.push_back(pm.reg_of.at(psrc_.stage_refs.back()[w]));
  if (semi && aggt_.kbits) {
    pp.semi_kbits = semi_all.as<uint32_t>();
    pp.semi_kmin = aggt_.kmin;
    pp.semi_krange = aggt_.krange;
    pp.semi_key_reg = p_out[0];
  } else if (semi) {
    pp.semi_bloom = semi_all.as<uint32_t>();
    pp.semi_words = bloom_words;
    pp.semi_shift = aggt_.bloom_shift;
    pp.semi_key_reg = p_out[0];
  }
  auto pfeed = open_feed(*psrc_.scan, file_cols_of(psrc_, pm));
  std::vector<DevCols> joined_parts;  // no-aggregate results
  ScanProgram pack{};  // bit-packed shuffle rows (pack_n > 0), set up below
  auto consume_materialised = [&](const BatchView& v, int ncols, cudaStream_t cs = nullptr) {
    // v: segments whose columns are p_out order (key first), or one bit-packed word per row.
    // cs: the aux stream of the chunked pipeline (ordered after the table insert already)
    if (!cs) join_build();
    if (agg_) {
      ScanProgram p = batch_program(ncols);
      p.sink = grouped_ ? SINK_PROBE : SINK_PROBE_GLOBAL;
      p.agg = aggt_;
      // received rows already passed the screen (the rank table still needs its bitmap: slots)
      if (semi && !aggt_.krank) p.agg.bloom = nullptr, p.agg.kbits = nullptr;
      p.key_reg = 0;
      p.n_sum = static_cast<int>(probe_sum_wire.size());
      for (int s = 0; s < p.n_sum; ++s) p.sum_reg[s] = 1 + s;
      if (pack.pack_n) {  // unpack register 0 into 1..n: key, sums
        p.unpack_n = pack.pack_n;
        for (int k = 0; k < pack.pack_n; ++k) {
          p.pack_min[k] = pack.pack_min[k];
          p.pack_shift[k] = pack.pack_shift[k];
          p.pack_mask[k] = pack.pack_mask[k];
        }
        p.n_regs = 1 + pack.pack_n;
        p.key_reg = 1;
        for (int s = 0; s < p.n_sum; ++s) p.sum_reg[s] = 2 + s;
      }
      if (!grouped_) {
        p.global_acc = global_acc_.as<unsigned long long>();
        for (int s = 0; s < p.n_sum; ++s) p.global_float[1 + s] = aggt_.ps_float[s];
        for (int b = 0; b < aggt_.nbs; ++b) p.global_float[1 + p.n_sum + b] = aggt_.bs_float[b];
      }
      run_scan(p, v, false, cs);
    } else {
      // compact, then expanding join against the final CSR table
      DevCols c = alloc_cols(ncols, std::max<uint64_t>(v.rows, 1));
      ScanProgram p = batch_program(ncols);
      p.n_early = ncols;
      std::vector<int> regs(ncols);
      std::iota(regs.begin(), regs.end(), 0);
      materialize_into(c, p, v, regs, -1, nullptr);
      const uint64_t n = read_count(c);
      DevBuf counts(ctx_.pool, (n + 1) * 4, ctx_.compute), offs(ctx_.pool, (n + 1) * 4, ctx_.compute);
      PSG_CUDA(cudaMemsetAsync(counts.p, 0, (n + 1) * 4, ctx_.compute));
      launch_expand_count(final_table->dev, c.cols[0].as<uint64_t>(), n, counts.as<uint32_t>(), ctx_.compute);
      size_t tb = exclusive_scan_u32(nullptr, nullptr, n + 1, nullptr, 0, ctx_.compute);
      DevBuf tmp(ctx_.pool, tb, ctx_.compute);
      exclusive_scan_u32(counts.as<uint32_t>(), offs.as<uint32_t>(), n + 1, tmp.p, tb, ctx_.compute);
      uint32_t total = 0;
      PSG_CUDA(cudaMemcpyAsync(&total, offs.as<uint32_t>() + n, 4, cudaMemcpyDeviceToHost, ctx_.compute));
      PSG_CUDA(cudaStreamSynchronize(ctx_.compute));
      const int np = final_table->dev.npayload;
      DevCols j = alloc_cols(np + ncols, std::max<uint64_t>(total, 1));
      std::vector<const uint64_t*> pc;
      std::vector<uint64_t*> oc;
      for (int q = 0; q < ncols; ++q) pc.push_back(c.cols[q].as<uint64_t>());
      for (int q = 0; q < np + ncols; ++q) oc.push_back(j.cols[q].as<uint64_t>());
      launch_expand_write(final_table->dev, c.cols[0].as<uint64_t>(), n, offs.as<uint32_t>(), pc.data(), ncols, oc.data(),
                          ctx_.compute);
      j.rows = total;
      joined_parts.push_back(std::move(j));
    }
  };

  if (p2p) {
    ScanProgram p = pp;
    p.sink = SINK_PROBE;
    p.agg = aggt_;
    p.agg.bloom = nullptr;
    p.remote = 1;
    p.peers = peers_dev.as<AggPeer>();
    p.nparts = nr;
    if (aggt_.bloom) {
      p.semi_bloom = semi_all.as<uint32_t>();
      p.semi_words = bloom_words;
      p.semi_shift = aggt_.bloom_shift;
      p.semi_key_reg = pm.reg_of.at(psrc_.stage_refs.back()[pkey]);
    }
    p.key_reg = pm.reg_of.at(psrc_.stage_refs.back()[pkey]);
    p.n_sum = static_cast<int>(probe_sum_wire.size());
    for (int s = 0; s < p.n_sum; ++s) p.sum_reg[s] = pm.reg_of.at(psrc_.stage_refs.back()[probe_sum_wire[s]]);
    BatchView v;
    while (pfeed->next(v)) {
      run_scan(p, v, staged_ != nullptr);
      pfeed->done();
      st_.ingest_bytes += v.bytes;
    }
    gpu_barrier();  // every rank's probe contributions landed before owners finalise
  } else if (slab_mode_) {
    // peer-slab shuffle: one fused kernel per probe batch - predicate, global semi-join screen,
    // late columns, owned rows probed in place, other rows stored into their owner's slab over
    // NVLink; then a device-side barrier and the owners fold what they received
    ScanProgram p = pp;
    p.sink = SINK_PROBE;
    p.staged_ok = 1;
    p.agg = aggt_;
    p.key_reg = pm.reg_of.at(psrc_.stage_refs.back()[pkey]);
    p.n_sum = static_cast<int>(probe_sum_wire.size());
    for (int k = 0; k < p.n_sum; ++k) p.sum_reg[k] = pm.reg_of.at(psrc_.stage_refs.back()[probe_sum_wire[k]]);
    apply_buckets(p);
    const int np = static_cast<int>(pneed.size());
    p.pack_n = np;
    for (int k = 0; k < np; ++k) {
      p.pack_reg[k] = p_out[k];
      p.pack_min[k] = slab_pack_.min[k];
      p.pack_shift[k] = slab_pack_.shift[k];
      p.pack_mask[k] = slab_pack_.mask[k];
    }
    p.slab = 1;
    p.slab_grec = slab_grec_.as<unsigned long long>();
    p.nparts = nr;
    p.self_rank = ctx_.rank;
    p.slab_cap = slab_cap_;
    unsigned long long* my_cnt = reinterpret_cast<unsigned long long*>(ctx_.symm + slab_cnt_off_);
    p.slab_cnt = my_cnt;
    // push (default): the probe kernel stores remote rows into the owner's inbox through NVLink,
    // so the transfer overlaps the scan and the owner-side fold reads local HBM; PSG_SLAB_PUSH=0
    // (pull): remote rows go to this rank's own outbox and the owner reads them over NVLink after
    // the barrier. SF100 A/B: N=2 3.02 / 3.02 ms (the fold is bound by its appends there), N=4
    // 2.05 / 2.11 ms (fold 0.14 / 0.18 ms: pulling from three peers is read-bound).
    static const bool push = [] {
      const char* e = std::getenv("PSG_SLAB_PUSH");
      return !(e && e[0] == '0');
    }();
    for (int d = 0; d < nr; ++d)
      p.slab_dst[d] = d == ctx_.rank ? nullptr
                      : push ? reinterpret_cast<uint64_t*>(ctx_.symm_peer[d] + slab_off_) + static_cast<uint64_t>(ctx_.rank) * slab_cap_
                             : reinterpret_cast<uint64_t*>(ctx_.symm + slab_off_) + static_cast<uint64_t>(d) * slab_cap_;
    // (the previous query's readers of these counters finished before this query's all-reduce)
    PSG_CUDA(cudaMemsetAsync(my_cnt, 0, static_cast<size_t>(nr) * 8, ctx_.compute));
    BatchView v;
    while (pfeed->next(v)) {
      run_scan(p, v, staged_ != nullptr);
      pfeed->done();
      st_.ingest_bytes += v.bytes;
    }
    pt.mark("  probe + slab stores", ctx_.compute);
    // PSG_CONSUME_PREFETCH=1: warm L2 with the rank records the owner-side fold reads while the
    // barrier waits for the other ranks (measured neutral at SF100 N=2: off)
    static const bool prefetch_env = [] {  // 1: bulk L2 prefetch, 2: evict-last loads
      const char* e = std::getenv("PSG_CONSUME_PREFETCH");
      return e && (e[0] == '1' || e[0] == '2');
    }();
    if (prefetch_env) launch_l2_prefetch(aggt_.krec, ((aggt_.krange + 63) / 64) * 16, ctx_.compute);
    gpu_barrier();  // every source's slab stores landed
    pt.mark("  barrier", ctx_.compute);
    SlabConsume c{};
    for (int r = 0; r < nr; ++r)
      c.src_rows[r] = r == ctx_.rank ? nullptr
                      : push ? reinterpret_cast<const uint64_t*>(ctx_.symm + slab_off_) + static_cast<uint64_t>(r) * slab_cap_
                             : reinterpret_cast<const uint64_t*>(ctx_.symm_peer[r] + slab_off_) + static_cast<uint64_t>(ctx_.rank) * slab_cap_;
    for (int r = 0; r < nr; ++r)
      c.src_cnt[r] = r == ctx_.rank ? nullptr
                                    : reinterpret_cast<const unsigned long long*>(ctx_.symm_peer[r] + slab_cnt_off_) + ctx_.rank;
    c.cap = slab_cap_;
    c.nsrc = nr;
    c.npack = np;
    for (int k = 0; k < np; ++k) {
      c.pshift[k] = slab_pack_.shift[k];
      c.pmask[k] = slab_pack_.mask[k];
      c.pmin[k] = slab_pack_.min[k];
    }
    c.bkt = p.bkt;
    c.fill = p.bkt_fill;
    c.bcap = p.bkt_cap;
    c.bsub_bits = p.bkt_sub_bits;
    for (int k = 0; k < kMaxSums; ++k) {
      c.bshift[k] = p.bkt_shift[k];
      c.bmask[k] = p.bkt_mask[k];
      c.bmin[k] = p.bkt_min[k];
    }
    c.ovf = p.bkt_ovf;
    c.ovf_count = p.bkt_ovf_count;
    c.ovf_cap = p.bkt_ovf_cap;
    slab_recv_ = DevBuf(ctx_.pool, 8, ctx_.compute);
    PSG_CUDA(cudaMemsetAsync(slab_recv_.p, 0, 8, ctx_.compute));
    c.received = slab_recv_.as<unsigned long long>();
    if (const char* e = std::getenv("PSG_SLAB_DIAG")) c.diag = std::atoi(e);
    launch_slab_consume(aggt_, c, ctx_.compute);
    pt.mark("  slab consume", ctx_.compute);
  } else if (nr == 1 && agg_ && !pdup) {
    ScanProgram p = pp;
    p.sink = grouped_ ? SINK_PROBE : SINK_PROBE_GLOBAL;
    p.staged_ok = 1;  // PSTO batches / staged images: 16-byte aligned chunks with tail padding
    p.agg = aggt_;
    p.key_reg = pm.reg_of.at(psrc_.stage_refs.back()[pkey]);
    p.n_sum = static_cast<int>(probe_sum_wire.size());
    for (int s = 0; s < p.n_sum; ++s) p.sum_reg[s] = pm.reg_of.at(psrc_.stage_refs.back()[probe_sum_wire[s]]);
    if (!grouped_) {
      p.global_acc = global_acc_.as<unsigned long long>();
      for (int s = 0; s < p.n_sum; ++s) p.global_float[1 + s] = aggt_.ps_float[s];
      for (int b = 0; b < aggt_.nbs; ++b) p.global_float[1 + p.n_sum + b] = aggt_.bs_float[b];
    }
    if (bucket_mode_) apply_buckets(p);
    // PSG_SLAB_FAKE=1: the peer-slab data path on one GPU, pretending to be rank 0 of 2 - half the
    // keys "remote": packed into a local outbox by the probe kernel and folded back by the
    // owner-side kernel - so the N > 1 kernels can be profiled with ncu and parity-tested in a
    // single process.
    DevBuf fake_out, fake_cnt;
    static const bool fake = [] {
      const char* e = std::getenv("PSG_SLAB_FAKE");
      return e && e[0] == '1';
    }();
    if (fake && bucket_mode_ && aggt_.krec && pneed.size() >= 2 && pneed.size() <= 4) {
      std::vector<int64_t> lo(pneed.size(), INT64_MAX), hi(pneed.size(), INT64_MIN);
      for (size_t k = 0; k < pneed.size(); ++k) {
        long long a = LLONG_MAX, b = LLONG_MIN;
        zone_range(psrc_.scan->paths, psrc_.proj.file_idx[psrc_.stage_refs.back()[pneed[k]].idx], a, b);
        lo[k] = a, hi[k] = b;
      }
      const PackLayout L = plan_pack(lo.data(), hi.data(), static_cast<int>(pneed.size()));
      uint64_t rows = 0;
      for (const auto& path : psrc_.scan->paths) rows += ctx_.footers.get(path)->total_rows();
      if (L.fits && L.bits < 64) {
        fake_out = DevBuf(ctx_.pool, (std::max<uint64_t>(rows, 1) + kSlabChunkSlack) * 8, ctx_.compute);
        fake_cnt = DevBuf(ctx_.pool, 16, ctx_.compute);
        PSG_CUDA(cudaMemsetAsync(fake_cnt.p, 0, 16, ctx_.compute));
        p.slab = 1;
        p.nparts = 2;
        p.self_rank = 0;
        p.slab_cap = std::max<uint64_t>(rows, 1) + kSlabChunkSlack;
        p.slab_cnt = fake_cnt.as<unsigned long long>();
        p.slab_dst[1] = fake_out.as<uint64_t>();
        p.semi_kbits = aggt_.kbits;
        p.semi_kmin = aggt_.kmin;
        p.semi_krange = aggt_.krange;
        p.semi_key_reg = p.key_reg;
        p.pack_n = static_cast<int>(pneed.size());
        for (size_t k = 0; k < pneed.size(); ++k) {
          p.pack_reg[k] = pm.reg_of.at(psrc_.stage_refs.back()[pneed[k]]);
          p.pack_min[k] = L.min[k];
          p.pack_shift[k] = L.shift[k];
          p.pack_mask[k] = L.mask[k];
        }
      }
    }
    BatchView v;
    while (pfeed->next(v)) {
      run_scan(p, v, staged_ != nullptr);
      pfeed->done();
      st_.ingest_bytes += v.bytes;
    }
    if (p.slab) {  // fake mode: fold the "remote" rows back in (the owner side, from the local outbox)
      SlabConsume c{};
      c.src_rows[1] = fake_out.as<uint64_t>();
      c.src_cnt[1] = fake_cnt.as<unsigned long long>() + 1;
      c.cap = p.slab_cap;
      c.nsrc = 2;
      c.npack = p.pack_n;
      for (int k = 0; k < p.pack_n; ++k) {
        c.pshift[k] = p.pack_shift[k];
        c.pmask[k] = p.pack_mask[k];
        c.pmin[k] = p.pack_min[k];
      }
      c.bkt = p.bkt;
      c.fill = p.bkt_fill;
      c.bcap = p.bkt_cap;
      c.bsub_bits = p.bkt_sub_bits;
      for (int k = 0; k < kMaxSums; ++k) {
        c.bshift[k] = p.bkt_shift[k];
        c.bmask[k] = p.bkt_mask[k];
        c.bmin[k] = p.bkt_min[k];
      }
      c.ovf = p.bkt_ovf;
      c.ovf_count = p.bkt_ovf_count;
      c.ovf_cap = p.bkt_ovf_cap;
      slab_recv_ = DevBuf(ctx_.pool, 8, ctx_.compute);
      PSG_CUDA(cudaMemsetAsync(slab_recv_.p, 0, 8, ctx_.compute));
      c.received = slab_recv_.as<unsigned long long>();
      launch_slab_consume(aggt_, c, ctx_.compute);
    }
  } else {
    uint64_t waves = pfeed->nbatches;
    if (nr > 1) {
      DevBuf wv(ctx_.pool, 8, ctx_.compute);
      PSG_CUDA(cudaMemcpyAsync(wv.p, &waves, 8, cudaMemcpyHostToDevice, ctx_.compute));
      PSG_NCCL(ncclAllReduce(wv.p, wv.p, 1, ncclUint64, ncclMax, ctx_.nccl, ctx_.compute));
      PSG_CUDA(cudaMemcpyAsync(&waves, wv.p, 8, cudaMemcpyDeviceToHost, ctx_.compute));
      PSG_CUDA(cudaStreamSynchronize(ctx_.compute));
    }
    // Bit-packed shuffle rows: the footer zone maps bound every shipped column; with the ranges
    // all-reduced (every rank packs and unpacks alike) a row whose fields fit in 64 bits travels
    // as ONE word (Q3: key 28 + price 17 + discount 4 bits instead of 3 x 64). PSG_PACK=0: off.
    static const bool pack_env = [] {
      const char* e = std::getenv("PSG_PACK");
      return !(e && std::string(e) == "0");
    }();
    if (nr > 1 && agg_ && jit_available() && pack_env && !pdup && pneed.size() <= static_cast<size_t>(kMaxOut)) {
      const size_t np = pneed.size();
      std::vector<long long> lohi(2 * np);
      for (size_t k = 0; k < np; ++k) {
        long long lo = LLONG_MAX, hi = LLONG_MIN;
        const ColRef ref = psrc_.stage_refs.back()[pneed[k]];
        if (ref.join >= 0 || psrc_.wire.fields[pneed[k]].type != LType::Int64) {
          lo = LLONG_MIN, hi = LLONG_MAX;  // not bounded by this scan's zone maps: never fits
        } else {
          zone_range(psrc_.scan->paths, psrc_.proj.file_idx[ref.idx], lo, hi);
        }
        lohi[k] = ~lo;  // one MAX all-reduce for both: max(~lo) = ~min(lo)
        lohi[np + k] = hi;
      }
      DevBuf red(ctx_.pool, 2 * np * 8, ctx_.compute);
      PSG_CUDA(cudaMemcpyAsync(red.p, lohi.data(), 2 * np * 8, cudaMemcpyHostToDevice, ctx_.compute));
      PSG_NCCL(ncclAllReduce(red.p, red.p, 2 * np, ncclInt64, ncclMax, ctx_.nccl, ctx_.compute));
      PSG_CUDA(cudaMemcpyAsync(lohi.data(), red.p, 2 * np * 8, cudaMemcpyDeviceToHost, ctx_.compute));
      PSG_CUDA(cudaStreamSynchronize(ctx_.compute));
      std::vector<int64_t> plo(np), phi(np);
      for (size_t k = 0; k < np; ++k) plo[k] = ~lohi[k], phi[k] = lohi[np + k];
      const PackLayout L = plan_pack(plo.data(), phi.data(), static_cast<int>(np));
      const bool fits = L.fits;
      for (size_t k = 0; k < np; ++k) {
        pack.pack_min[k] = L.min[k];
        pack.pack_shift[k] = L.shift[k];
        pack.pack_mask[k] = L.mask[k];
      }
      if (fits && np > 1) {
        pack.pack_n = static_cast<int>(np);
        pp.pack_n = pack.pack_n;
        for (size_t k = 0; k < np; ++k) {
          pp.pack_reg[k] = p_out[k];
          pp.pack_min[k] = pack.pack_min[k];
          pp.pack_shift[k] = pack.pack_shift[k];
          pp.pack_mask[k] = pack.pack_mask[k];
        }
      }
    }
    // When rows cannot be packed, the rows this rank owns are probed and aggregated in place by
    // the partitioning scan itself: only rows owned by other ranks are materialised and shuffled.
    // (Measured at N=2: packing alone 6.39 ms, owner probe alone 6.62, both 6.98, neither 6.86 -
    // the in-kernel probe slows the scan more than it saves once rows are one word.)
    // PSG_SELF_PROBE=0 turns it off (A/B measurements).
    static const bool self_probe_env = [] {
      const char* e = std::getenv("PSG_SELF_PROBE");
      return !(e && std::string(e) == "0");
    }();
    if (nr > 1 && agg_ && grouped_ && jit_available() && self_probe_env && pack.pack_n == 0 && !pdup &&
        !aggt_.krank) {
      join_build();  // the scan itself probes this rank's table
      pp.self_probe = 1;
      pp.self_rank = ctx_.rank;
      pp.agg = aggt_;
      pp.agg.bloom = nullptr;  // the semi-join screen already tested the owner's (= our) filter
      pp.key_reg = p_out[0];
      pp.n_sum = static_cast<int>(probe_sum_wire.size());
      for (int k = 0; k < pp.n_sum; ++k) pp.sum_reg[k] = p_out[1 + k];
    }
    const std::vector<int> mat_out = pack.pack_n ? std::vector<int>{p_out[0]} : p_out;
    const KeyField kf = pack.pack_n ? KeyField{pack.pack_min[0], pack.pack_mask[0], 0} : KeyField{0, 0, 0};
    // Staged probe side at N > 1: the scan is cut into K chunks of whole segments; chunk k+1's
    // scan/screen/partition kernel runs on the compute stream while chunk k is exchanged (counts,
    // scatter, NCCL send/recv) and consumed into the table on the aux stream, so the shuffle and
    // the table probes could overlap the scan. K is the same on every rank (collective order).
    // Parity-green (scripts/mgpu_check.py staged runs) but measured slower, so off by default:
    // N=2 SF100 5.98 ms unchunked vs 7.0-7.3 (K=2, 4) and 6.85 (K=8) - the persistent scan grid
    // holds every SM until it ends, so the NCCL and consume kernels on the aux stream wait for it
    // anyway, and each chunk adds a count all-gather, a host sync and a send/recv round.
    // PSG_PROBE_CHUNKS: K (default 1 = off).
    static const int probe_chunks = [] {
      const char* e = std::getenv("PSG_PROBE_CHUNKS");
      return e ? std::max(1, std::atoi(e)) : 1;
    }();
    const std::vector<Segment>* hsegs = pfeed->host_segments();
    if (nr > 1 && agg_ && hsegs != nullptr && waves == 1 && probe_chunks > 1 && !pdup) {
      const int K = probe_chunks;
      BatchView whole;
      if (pfeed->next(whole)) st_.ingest_bytes += whole.bytes;
      std::vector<std::vector<Segment>> parts(K);
      uint64_t tot = 0, acc = 0;
      for (const auto& sg : *hsegs) tot += sg.rows;
      int k = 0;
      for (const auto& sg : *hsegs) {
        while (k < K - 1 && acc >= tot * static_cast<uint64_t>(k + 1) / K) ++k;
        parts[k].push_back(sg);
        acc += sg.rows;
      }
      struct Evs {
        std::vector<cudaEvent_t> e;
        Evs(size_t n, unsigned flags) : e(n) {
          for (auto& x : e) cudaEventCreateWithFlags(&x, flags);
        }
        ~Evs() {
          for (auto x : e) cudaEventDestroy(x);
        }
      };
      Evs done(K + 1, cudaEventDisableTiming), t0(K, cudaEventDefault), t1(K, cudaEventDefault);
      std::vector<DevBuf> seg_hold(K), rholds(K);
      std::vector<BatchView> views(K);
      for (int c = 0; c < K; ++c) views[c] = upload_segments(parts[c], seg_hold[c]);
      std::vector<DevCols> mats;
      std::vector<DevBuf> pcs;
      std::vector<Received> recvs;
      mats.reserve(K), pcs.reserve(K), recvs.reserve(K);
      // the aux stream starts after everything queued so far (tables, filters, segment tables)
      PSG_CUDA(cudaEventRecord(done.e[K], ctx_.compute));
      PSG_CUDA(cudaStreamWaitEvent(ctx_.comm, done.e[K], 0));
      auto launch_chunk = [&](int c) {
        mats.push_back(alloc_cols(mat_out.size(), std::max<uint64_t>(views[c].rows, 1)));
        pcs.emplace_back(ctx_.pool, nr * 8, ctx_.compute);
        PSG_CUDA(cudaMemsetAsync(pcs[c].p, 0, nr * 8, ctx_.compute));
        PSG_CUDA(cudaEventRecord(t0.e[c], ctx_.compute));
        materialize_into(mats[c], pp, views[c], mat_out, p_out[0], &pcs[c], false, true);
        PSG_CUDA(cudaEventRecord(t1.e[c], ctx_.compute));
        PSG_CUDA(cudaEventRecord(done.e[c], ctx_.compute));
      };
      launch_chunk(0);
      for (int c = 0; c < K; ++c) {
        if (c + 1 < K) launch_chunk(c + 1);
        PSG_CUDA(cudaStreamWaitEvent(ctx_.comm, done.e[c], 0));
        recvs.push_back(exchange(mats[c], static_cast<int>(mat_out.size()), 0, pcs[c], views[c].nsegs > 0, kf, ctx_.comm));
        BatchView rv = upload_segments(recvs[c].segs, rholds[c], ctx_.comm);
        consume_materialised(rv, static_cast<int>(mat_out.size()), ctx_.comm);
      }
      PSG_CUDA(cudaEventRecord(done.e[K], ctx_.comm));
      PSG_CUDA(cudaStreamWaitEvent(ctx_.compute, done.e[K], 0));
      join_build();
      PSG_CUDA(cudaStreamSynchronize(ctx_.compute));
      for (int c = 0; c < K; ++c) {
        if (!views[c].nsegs) continue;
        float ms = 0;
        PSG_CUDA(cudaEventElapsedTime(&ms, t0.e[c], t1.e[c]));
        st_.probe_kernel_ms += ms;
        st_.probe_kernel_launches += 1;
      }
      st_.probe_kernel_bytes += whole.bytes;
      pt.mark("  probe chunks (scan | exchange + consume)", ctx_.compute);
      waves = 0;
    }
    for (uint64_t w = 0; w < waves; ++w) {
      BatchView v;
      const bool have = pfeed->next(v);
      DevCols mat = alloc_cols(mat_out.size(), std::max<uint64_t>(have ? v.rows : 1, 1));
      DevBuf pc(ctx_.pool, nr * 8, ctx_.compute);
      PSG_CUDA(cudaMemsetAsync(pc.p, 0, nr * 8, ctx_.compute));
      if (have && pdup) {
        mat = materialize_chain(psrc_, pm, v, mat_out);
        if (nr > 1) launch_part_hist(mat.cols[0].as<uint64_t>(), mat.rows, nr, pc.as<unsigned long long>(), ctx_.compute);
        pfeed->done();
        st_.ingest_bytes += v.bytes;
      } else if (have) {
        materialize_into(mat, pp, v, mat_out, p_out[0], &pc, staged_ != nullptr, true);
        pfeed->done();
        st_.ingest_bytes += v.bytes;
      }
      pt.mark("  probe materialize", ctx_.compute);
      if (nr > 1) {
        Received r = exchange(mat, static_cast<int>(mat_out.size()), 0, pc, have, kf);
        DevBuf holder;
        BatchView rv = upload_segments(r.segs, holder);
        pt.mark("  probe exchange", ctx_.compute);
        consume_materialised(rv, static_cast<int>(mat_out.size()));
        PSG_CUDA(cudaStreamSynchronize(ctx_.compute));
        pt.mark("  probe consume", ctx_.compute);
      } else {
        const uint64_t n = read_count(mat);
        Segment sg;
        std::memset(&sg, 0, sizeof sg);
        for (size_t c = 0; c < p_out.size(); ++c) sg.col[c] = mat.cols[c].as<uint64_t>();
        sg.rows = n;
        DevBuf holder;
        std::vector<Segment> one;
        if (n) one.push_back(sg);
        BatchView rv = upload_segments(one, holder);
        consume_materialised(rv, static_cast<int>(p_out.size()));
        PSG_CUDA(cudaStreamSynchronize(ctx_.compute));
      }
    }
  }
  join_build();
  PSG_CUDA(cudaStreamSynchronize(ctx_.compute));
  st_.storage_phase_s = secs_since(t_storage);

  pt.mark("probe side", ctx_.compute);
  // ---------------- finalize ----------------
  if (agg_) {
    pt.mark("  pre finalize", ctx_.compute);
    if (grouped_) finalize_grouped(out, want_rows);
    else finalize_global(out);
  } else {
    const int nc = static_cast<int>(result_schema_.size());
    uint64_t total = 0;
    for (auto& j : joined_parts) total += j.rows;
    out.nrows = total;
    if (want_rows) {
      uint64_t* dst = out.mutable_rows(total * nc);
      uint64_t at = 0;
      for (auto& j : joined_parts) {
        if (!j.rows) continue;
        DevBuf rows(ctx_.pool, j.rows * nc * 8, ctx_.compute);
        // joined columns are [build payload..., probe key, probe others...]; restore the probe
        // side's wire order (payload ++ probe wire, ops.cpp:193-200)
        std::vector<const uint64_t*> cols;
        const int npay = nc - static_cast<int>(psrc_.wire.size());
        for (int c = 0; c < npay; ++c) cols.push_back(j.cols[c].as<uint64_t>());
        for (size_t w = 0; w < psrc_.wire.size(); ++w) {
          const int at = static_cast<int>(std::find(pneed.begin(), pneed.end(), static_cast<int>(w)) - pneed.begin());
          cols.push_back(j.cols[npay + at].as<uint64_t>());
        }
        launch_rows_from_cols(cols.data(), nc, j.rows, rows.as<uint64_t>(), ctx_.compute);
        PSG_CUDA(cudaMemcpyAsync(dst + at * nc, rows.p, j.rows * nc * 8, cudaMemcpyDeviceToHost, ctx_.compute));
        PSG_CUDA(cudaStreamSynchronize(ctx_.compute));
        at += j.rows;
      }
      st_.result_bytes += total * nc * 8;
    }
  }
  if (!lt_flags_.empty()) enqueue_lt_flags();
  PSG_CUDA(cudaStreamSynchronize(ctx_.compute));
  PSG_CUDA(cudaGetLastError());
  if (!lt_flags_.empty()) check_lt_flags();
  pt.mark("finalize", ctx_.compute);
  PSG_CUDA(cudaEventRecord(ev1, ctx_.compute));
  PSG_CUDA(cudaEventSynchronize(ev1));
  float dms = 0;
  PSG_CUDA(cudaEventElapsedTime(&dms, ev0, ev1));
  cudaEventDestroy(ev0);
  cudaEventDestroy(ev1);
  st_.device_ms = dms;
  resolve_timed();
  sum_exchange_time();
  if (session_) {
    session_->check_inflate();
    st_.h2d_bytes = session_->h2d_bytes;
  }
  if (session_ && session_->ingest) st_.io_wait_s = session_->ingest->wait_s();
  if (timeline) {
    session_.reset();  // drains the streams and the I/O threads first
    timeline->dump(std::getenv("PSG_TIMELINE"), ctx_.rank);
  }
  st_.jit_compiles = jit_stats().compiles - jit0_;
  st_.result_rows = out.nrows;
  st_.runtime_s = secs_since(t0);
  st_.peak_bytes = ctx_.pool.peak();
  st_.kernel_launches = kernel_launch_count() - launches0_;
  out.stats = st_;
  return out;
}

// ------------------------------------------------------------------------- local plans
/// Scan -> filter -> replicated local joins -> global aggregate, with no exchange: the Q6-analog
/// plan family. The reference's execute_plan rejects plans without a shuffled
/// join (pipeline.cpp:334-335), so this is an extension entry (psg_execute_local); per node it
/// returns one unmerged partial row [rows, sums...] exactly like a global aggregate of
/// execute_plan (pipeline.cpp:277-281, 892-897).
ResultRows Execution::run_local() {
  const auto t0 = Clock::now();
  launches0_ = kernel_launch_count();
  jit0_ = jit_stats().compiles;
  ctx_.pool.reset_peak();
  BudgetScope budget_scope(ctx_.pool, plan_.memory_budget_bytes);
  cudaEvent_t ev0, ev1;
  PSG_CUDA(cudaEventCreate(&ev0));
  PSG_CUDA(cudaEventCreate(&ev1));
  PSG_CUDA(cudaEventRecord(ev0, ctx_.compute));
  plan_.validate();
  if (plan_.shuffle_join()) throw InvalidInput("local plans have no shuffled join (use execute_plan)");
  if (!plan_.aggregate || !plan_.aggregate->group_by.empty())
    throw InvalidInput("local plans end in a global aggregate (no group_by)");
  // the root: the one stream no join consumes (a scan, or the last replicated join)
  std::set<std::string> consumed;
  for (const auto& j : plan_.joins) consumed.insert(j.build), consumed.insert(j.probe);
  std::vector<std::string> roots;
  for (const auto& j : plan_.joins)
    if (!consumed.count(j.id)) roots.push_back(j.id);
  for (const auto& sc : plan_.scans)
    if (!sc.replicated && !consumed.count(sc.table)) roots.push_back(sc.table);
  if (roots.size() != 1) throw InvalidInput("a local plan needs exactly one root stream");
  psrc_ = make_source(plan_, ctx_.footers, roots[0]);
  agg_ = true;
  grouped_ = false;
  result_schema_.fields.push_back(Field{"rows", LType::Int64});
  for (const auto& c : plan_.aggregate->sums) {
    const size_t w = psrc_.wire.require(c);
    result_schema_.fields.push_back(Field{"sum_" + psrc_.wire.fields[w].name, psrc_.wire.fields[w].type});
    sum_order.push_back({1, static_cast<int>(probe_sum_wire.size())});
    probe_sum_wire.push_back(static_cast<int>(w));
  }
  if (probe_sum_wire.size() > static_cast<size_t>(kMaxSums)) throw InvalidInput("too many aggregate sums");
  ResultRows out;
  out.schema = result_schema_;
  std::vector<int> need = probe_sum_wire;
  if (need.empty() && psrc_.scan->predicate.empty()) need.push_back(0);  // a column to count rows over
  RegMap pm = analyse(psrc_, need, -1, true);
  for (size_t j = 0; j < psrc_.chain.size(); ++j) psrc_.chain[j].needed_payload = pm.payload_cols[j];
  {  // one ingest session: the replicated scans of the chain, then the root scan
    std::vector<std::pair<const ScanNode*, std::vector<int>>> scans;
    for (size_t j = 0; j < psrc_.chain.size(); ++j) {
      LocalJoinDef& lj = psrc_.chain[j];
      SourceDef rs;
      rs.scan = lj.scan;
      rs.proj = lj.proj;
      rs.wire = lj.proj.schema;
      std::vector<ColRef> refs;
      for (size_t i = 0; i < rs.wire.size(); ++i) refs.push_back({-1, static_cast<int>(i)});
      rs.stage_refs.push_back(refs);
      std::vector<int> needed{lj.key_idx};
      for (int p : pm.payload_cols[j]) needed.push_back(lj.payload_idx[p]);
      RegMap rm = analyse(rs, needed, -1, false);
      scans.push_back({lj.scan, file_cols_of(rs, rm)});
    }
    scans.push_back({psrc_.scan, file_cols_of(psrc_, pm)});
    const uint64_t ht_reserve = plan_.ht_estimate_bytes ? plan_.ht_estimate_bytes : plan_.memory_budget_bytes / 4;
    session_ = std::make_unique<StreamSession>(ctx_, scans, plan_.memory_budget_bytes, ht_reserve);
  }
  build_local_tables();
  const bool pdup = dup_chain(psrc_);
  global_acc_ = DevBuf(ctx_.pool, (2 * kMaxSums + 1) * 8, ctx_.compute);
  PSG_CUDA(cudaMemsetAsync(global_acc_.p, 0, (2 * kMaxSums + 1) * 8, ctx_.compute));
  ScanProgram p = base_program(psrc_, pm, true);
  p.sink = SINK_AGG_SCAN;
  p.n_sum = static_cast<int>(probe_sum_wire.size());
  for (int k = 0; k < p.n_sum; ++k) {
    p.sum_reg[k] = pm.reg_of.at(psrc_.stage_refs.back()[probe_sum_wire[k]]);
    p.global_float[1 + k] = psrc_.wire.fields[probe_sum_wire[k]].type == LType::Float64;
  }
  p.global_acc = global_acc_.as<unsigned long long>();
  auto feed = open_feed(*psrc_.scan, file_cols_of(psrc_, pm));
  BatchView v;
  while (feed->next(v)) {
    if (pdup) {  // expanding local joins: compact + expand, then sum the materialised rows
      std::vector<int> regs;
      for (int w : need) regs.push_back(pm.reg_of.at(psrc_.stage_refs.back()[w]));
      DevCols mat = materialize_chain(psrc_, pm, v, regs);
      ScanProgram q;
      std::memset(&q, 0, sizeof q);
      q.n_in = static_cast<int>(regs.size());
      q.n_early = q.n_in;
      q.n_regs = std::max(1, q.n_in);
      q.part_key_reg = -1;
      q.key_reg = -1;
      q.sink = SINK_AGG_SCAN;
      q.n_sum = p.n_sum;
      for (int k = 0; k < q.n_sum; ++k) {
        q.sum_reg[k] = k;  // need[k] == probe_sum_wire[k]
        q.global_float[1 + k] = p.global_float[1 + k];
      }
      q.global_acc = p.global_acc;
      Segment sg;
      std::memset(&sg, 0, sizeof sg);
      for (size_t c = 0; c < regs.size(); ++c) sg.col[c] = mat.cols[c].as<uint64_t>();
      sg.rows = mat.rows;
      std::vector<Segment> one;
      if (sg.rows) one.push_back(sg);
      DevBuf holder;
      BatchView mv = upload_segments(one, holder);
      run_scan(q, mv, false);
      PSG_CUDA(cudaStreamSynchronize(ctx_.compute));
    } else {
      run_scan(p, v, false);
    }
    feed->done();
    st_.ingest_bytes += v.bytes;
  }
  finalize_global(out);
  if (!lt_flags_.empty()) enqueue_lt_flags();
  PSG_CUDA(cudaEventRecord(ev1, ctx_.compute));
  PSG_CUDA(cudaEventSynchronize(ev1));
  if (!lt_flags_.empty()) check_lt_flags();
  float dms = 0;
  PSG_CUDA(cudaEventElapsedTime(&dms, ev0, ev1));
  cudaEventDestroy(ev0);
  cudaEventDestroy(ev1);
  st_.device_ms = dms;
  resolve_timed();
  session_->check_inflate();
  st_.h2d_bytes = session_->h2d_bytes;
  if (session_->ingest) st_.io_wait_s = session_->ingest->wait_s();
  st_.jit_compiles = jit_stats().compiles - jit0_;
  st_.result_rows = out.nrows;
  st_.runtime_s = secs_since(t0);
  st_.peak_bytes = ctx_.pool.peak();
  st_.kernel_launches = kernel_launch_count() - launches0_;
  out.stats = st_;
  return out;
}

std::vector<std::pair<const ScanNode*, std::vector<int>>> Execution::scan_list(const RegMap& bm, const RegMap& pm) {
  std::vector<std::pair<const ScanNode*, std::vector<int>>> scans;
  for (int side = 0; side < 2; ++side) {
    SourceDef& s = side == 0 ? bsrc_ : psrc_;
    const RegMap& m = side == 0 ? bm : pm;
    for (size_t j = 0; j < s.chain.size(); ++j) {
      LocalJoinDef& lj = s.chain[j];
      SourceDef rs;
      rs.scan = lj.scan;
      rs.proj = lj.proj;
      rs.wire = lj.proj.schema;
      std::vector<ColRef> refs;
      for (size_t i = 0; i < rs.wire.size(); ++i) refs.push_back({-1, static_cast<int>(i)});
      rs.stage_refs.push_back(refs);
      std::vector<int> needed{lj.key_idx};
      for (int p : m.payload_cols[j]) needed.push_back(lj.payload_idx[p]);
      RegMap rm = analyse(rs, needed, -1, false);
      scans.push_back({lj.scan, file_cols_of(rs, rm)});
    }
  }
  scans.push_back({bsrc_.scan, file_cols_of(bsrc_, bm)});
  scans.push_back({psrc_.scan, file_cols_of(psrc_, pm)});
  return scans;
}

ResultRows Execution::run_ingest_only() {
  const auto t0 = Clock::now();
  compile();
  const int bkey = static_cast<int>(bsrc_.wire.require(shuffle_->build_key));
  const int pkey = static_cast<int>(psrc_.wire.require(shuffle_->probe_key));
  std::vector<int> bneed{bkey}, pneed{pkey};
  if (agg_) {
    for (int w : build_sum_wire) bneed.push_back(w);
    for (int w : probe_sum_wire) pneed.push_back(w);
  } else {
    for (size_t i = 0; i < bsrc_.wire.size(); ++i)
      if (static_cast<int>(i) != bkey) bneed.push_back(static_cast<int>(i));
    for (size_t i = 0; i < psrc_.wire.size(); ++i)
      if (static_cast<int>(i) != pkey) pneed.push_back(static_cast<int>(i));
  }
  RegMap bm = analyse(bsrc_, bneed, -1, true);
  RegMap pm = analyse(psrc_, pneed, pkey, true);
  for (size_t j = 0; j < bsrc_.chain.size(); ++j) bsrc_.chain[j].needed_payload = bm.payload_cols[j];
  for (size_t j = 0; j < psrc_.chain.size(); ++j) psrc_.chain[j].needed_payload = pm.payload_cols[j];
  session_ = std::make_unique<StreamSession>(ctx_, scan_list(bm, pm), 0, 0);
  for (size_t i = 0; i < session_->batches.size(); ++i) {
    BatchView v;
    session_->stage(i, v);
    st_.ingest_bytes += v.bytes;
    session_->release();
  }
  PSG_CUDA(cudaStreamSynchronize(ctx_.compute));
  session_->check_inflate();
  ResultRows out;
  st_.h2d_bytes = session_->h2d_bytes;
  if (session_->ingest) st_.io_wait_s = session_->ingest->wait_s();
  st_.runtime_s = secs_since(t0);
  out.stats = st_;
  return out;
}

void Execution::stage(Staged& st) {
  compile();
  const int bkey = static_cast<int>(bsrc_.wire.require(shuffle_->build_key));
  const int pkey = static_cast<int>(psrc_.wire.require(shuffle_->probe_key));
  std::vector<int> bneed{bkey}, pneed{pkey};
  if (agg_) {
    for (int w : build_sum_wire) bneed.push_back(w);
    for (int w : probe_sum_wire) pneed.push_back(w);
  } else {
    for (size_t i = 0; i < bsrc_.wire.size(); ++i)
      if (static_cast<int>(i) != bkey) bneed.push_back(static_cast<int>(i));
    for (size_t i = 0; i < psrc_.wire.size(); ++i)
      if (static_cast<int>(i) != pkey) pneed.push_back(static_cast<int>(i));
  }
  RegMap bm = analyse(bsrc_, bneed, -1, true);
  RegMap pm = analyse(psrc_, pneed, pkey, true);
  const auto scans = scan_list(bm, pm);
  for (auto& [scan, fcols] : scans) {
    const std::string key = scan_key(*scan, fcols);
    if (st.scans.count(key)) continue;
    ScanBatches sb = plan_batches(ctx_.footers, *scan, fcols, 0, ctx_.batch_bytes);
    StagedScan& ss = st.scans[key];
    // block codec: compressed images land in a transient buffer and are inflated into `data`
    uint64_t data_bytes = 0, wire_bytes = 0;
    for (auto& b : sb.batches) {
      data_bytes += b.inflate ? b.dbytes : b.bytes;
      wire_bytes += b.inflate ? b.bytes : 0;
    }
    ss.data = DevBuf(ctx_.pool, std::max<uint64_t>(data_bytes, 8), ctx_.compute);
    DevBuf wire, jobs_dev, err;
    if (wire_bytes) wire = DevBuf(ctx_.pool, wire_bytes, ctx_.compute);
    PSG_CUDA(cudaStreamSynchronize(ctx_.compute));
    std::vector<Segment> all;
    std::vector<InflateJob> jobs;
    const uint64_t slot_bytes = (std::max(sb.max_batch_bytes, ctx_.batch_bytes) + 4095) & ~4095ULL;
    if (!sb.batches.empty()) {
      const int threads = std::max(1, ctx_.io_threads);
      Ingest ing(ctx_, scan->paths, sb.batches, threads, slot_bytes, threads * 2 + 2);
      uint64_t woff = 0, doff = 0;
      for (size_t i = 0; i < sb.batches.size(); ++i) {
        const BatchPlan& b = sb.batches[i];
        uint8_t* dbase = ss.data.as<uint8_t>() + doff;
        uint8_t* base = b.inflate ? wire.as<uint8_t>() + woff : dbase;
        uint64_t nt = 0;
        auto segs = make_segments(b, dbase, nt);
        all.insert(all.end(), segs.begin(), segs.end());
        if (b.inflate) {
          auto bj = inflate_jobs(b, base, dbase);
          jobs.insert(jobs.end(), bj.begin(), bj.end());
        }
        ing.copy_to_device(i, base, nullptr, 0, ctx_.copy);
        st.h2d += b.bytes;
        woff += b.inflate ? b.bytes : 0;
        doff += b.inflate ? b.dbytes : b.bytes;
      }
      PSG_CUDA(cudaStreamSynchronize(ctx_.copy));
    }
    if (!jobs.empty()) {
      // one launch over every chunk of the scan: tens of thousands of concurrent decoders
      std::sort(jobs.begin(), jobs.end(), [](const InflateJob& a, const InflateJob& b) { return a.csize > b.csize; });
      jobs_dev = DevBuf(ctx_.pool, jobs.size() * sizeof(InflateJob), ctx_.compute);
      err = DevBuf(ctx_.pool, sizeof(unsigned int), ctx_.compute);
      PSG_CUDA(cudaMemcpyAsync(jobs_dev.p, jobs.data(), jobs.size() * sizeof(InflateJob), cudaMemcpyHostToDevice,
                               ctx_.compute));
      PSG_CUDA(cudaMemsetAsync(err.p, 0, sizeof(unsigned int), ctx_.compute));
      launch_inflate(jobs_dev.as<InflateJob>(), static_cast<uint32_t>(jobs.size()), err.as<unsigned int>(), ctx_.compute);
      unsigned int e = 0;
      PSG_CUDA(cudaMemcpyAsync(&e, err.p, sizeof e, cudaMemcpyDeviceToHost, ctx_.compute));
      PSG_CUDA(cudaStreamSynchronize(ctx_.compute));
      if (e) throw IoFailure("inflate failed");
    }
    const uint64_t T = static_cast<uint64_t>(scan_tile_rows());
    uint64_t tiles = 0;
    for (auto& s : all) {
      s.tile_begin = tiles;
      tiles += (s.rows + T - 1) / T;
    }
    ss.nsegs = static_cast<int>(all.size());
    ss.host_segs = all;
    ss.ntiles = tiles;
    ss.rows = sb.total_rows;
    ss.bytes = data_bytes;
    ss.payload = sb.total_scan;
    if (!all.empty()) {
      auto blob = pack_view(all, ss.tile_off);
      ss.segs = DevBuf(ctx_.pool, blob.size(), ctx_.compute);
      PSG_CUDA(cudaMemcpyAsync(ss.segs.p, blob.data(), blob.size(), cudaMemcpyHostToDevice, ctx_.compute));
      PSG_CUDA(cudaStreamSynchronize(ctx_.compute));
    }
    st.bytes += sb.total_scan;
  }
}

}  // namespace

ResultRows execute_plan(Ctx& ctx, const std::string& plan_json, const std::string& data_root, int mode, Staged* staged,
                        bool want_rows) {
  PSG_CUDA(cudaSetDevice(ctx.device));
  if (mode < 0 || mode > 3) throw InvalidInput("unknown execution mode");
  if (ctx.nranks > 1 && ctx.nccl == nullptr) throw InvalidInput("nranks > 1 needs psg_ctx_init_comm first");
  // a bucket-overflow-list overflow re-runs the query without buckets, a key-bitmap build that
  // does not apply re-runs it on the materialising build path (every rank takes the same decision:
  // both come from all-reduced values)
  auto with_retry = [&](auto&& once) {
    struct Flags {
      Ctx& c;
      ~Flags() { c.no_buckets = c.no_keybits = false; }
    } flags{ctx};
    for (int attempt = 0;; ++attempt) {
      try {
        return once();
      } catch (const BucketOverflow&) {
        if (ctx.no_buckets || attempt >= 2) throw;
        ctx.no_buckets = true;
      } catch (const KeybitsRetry&) {
        if (ctx.no_keybits || attempt >= 2) throw;
        ctx.no_keybits = true;
      }
    }
  };
  if (staged) {
    return with_retry([&] {
      Execution ex(ctx, staged->plan_json, staged->data_root, mode, staged);
      return ex.run(want_rows);
    });
  }
  if (mode == PSG_MODE_OVERLAPPED) {
    return with_retry([&] {
      Execution ex(ctx, plan_json, data_root, mode, nullptr);
      return ex.run(want_rows);
    });
  }
  // Phase-sequential modes: storage phase materialises every needed chunk in HBM, then the
  // network/compute phase runs over the staged images (run_phased, pipeline.cpp:506-556).
  const auto t0 = Clock::now();
  // Phase-sequential modes materialise every needed chunk: under a plan budget smaller than the
  // staged input this raises MemoryExceeded, like the reference's blocking reader (scan.cpp:289-292).
  const QueryPlan budget_plan = QueryPlan::from_json_text(plan_json, data_root, ctx.rank, ctx.nranks);
  if (budget_plan.memory_budget_bytes) ctx.pool.set_budget(ctx.pool.used() + budget_plan.memory_budget_bytes);
  std::unique_ptr<Staged> st;
  try {
    st.reset(stage_plan(ctx, plan_json, data_root));
  } catch (...) {
    ctx.pool.set_budget(0);
    throw;
  }
  ctx.pool.set_budget(0);
  const double storage = secs_since(t0);
  ResultRows r = with_retry([&] {
    Execution ex(ctx, plan_json, data_root, mode, st.get());
    return ex.run(want_rows);
  });
  r.stats.storage_phase_s = storage;
  r.stats.network_phase_s = r.stats.runtime_s;
  r.stats.runtime_s = secs_since(t0);
  r.stats.ingest_bytes = st->bytes;
  r.stats.h2d_bytes = st->h2d;
  return r;
}

ResultRows execute_local(Ctx& ctx, const std::string& plan_json, const std::string& data_root, int mode) {
  PSG_CUDA(cudaSetDevice(ctx.device));
  if (mode < 0 || mode > 3) throw InvalidInput("unknown execution mode");
  // a local semi-join bitmap that found duplicate keys re-runs on the materialising path
  try {
    Execution ex(ctx, plan_json, data_root, mode, nullptr);
    return ex.run_local();
  } catch (const KeybitsRetry&) {
    struct Flag {
      Ctx& c;
      ~Flag() { c.no_keybits = false; }
    } flag{ctx};
    ctx.no_keybits = true;
    Execution ex(ctx, plan_json, data_root, mode, nullptr);
    return ex.run_local();
  }
}

Staged* stage_plan(Ctx& ctx, const std::string& plan_json, const std::string& data_root) {
  PSG_CUDA(cudaSetDevice(ctx.device));
  auto st = std::make_unique<Staged>();
  st->plan_json = plan_json;
  st->data_root = data_root;
  Execution ex(ctx, plan_json, data_root, PSG_MODE_BLOCKING, nullptr);
  ex.stage(*st);
  return st.release();
}

void free_staged(Staged* s) { delete s; }

ResultRows ingest_only(Ctx& ctx, const std::string& plan_json, const std::string& data_root) {
  PSG_CUDA(cudaSetDevice(ctx.device));
  Execution ex(ctx, plan_json, data_root, PSG_MODE_OVERLAPPED, nullptr);
  return ex.run_ingest_only();
}

}  // namespace psg
