// The distributed-join microbenchmark on B200s: the reference's symmetric-repartitioning hash join
// in its four scheduling variants (run_join, /root/reference/proj/src/join.cpp:55-124 plans,
// :158-437 execution; harness run_sim_join, join_harness.cpp:43-97), re-designed for CUDA streams.
//
// Every variant runs the same operators - per wave: partition (destination histogram + scatter
// into destination-major columnar slabs), size exchange (NCCL all-gather of the count matrix),
// shuffle (grouped ncclSend/ncclRecv), then one CSR hash-table build over all received build rows
// and an expanding probe per received probe wave (payload ++ probe columns, ops.cpp:193-200). They
// differ only in how the steps are ordered over streams and where the host waits, which is what
// the paper measures:
//   * a "data-dependent" step (concat, partition, sizes, build, probe - OpDesc::data_dependent,
//     exec.cpp:54-66) makes the control thread wait for its stream (cudaStreamSynchronize);
//   * the shuffle is asynchronous (NCCL on the communication stream, ordered by events), so the
//     next wave's partition on another stream overlaps the transfer;
//   * deferred: wave w's probe is issued as the first step of wave w + k on its stream, so its
//     synchronising probe lands after the next wave's shuffle has been front-loaded.
// Blocking = whole-table phases on one stream with a fresh cudaMalloc/cudaFree per buffer (the
// reference's per-allocation pool mode); BlockingOpt = the same schedule on the pooled allocator.
#include <algorithm>
#include <chrono>
#include <cstring>
#include <numeric>

#include "engine.hpp"
#include "shuffle_plan.hpp"

#define PSG_NCCL_J(call)                                                                              \
  do {                                                                                                \
    ncclResult_t r_ = (call);                                                                         \
    if (r_ != ncclSuccess) throw ::psg::Error(PSG_ERR_NCCL, std::string("nccl: ") + ncclGetErrorString(r_)); \
  } while (0)

namespace psg {

// ------------------------------------------------------------------------------ the schedules
std::vector<JoinStep> join_schedule(int variant, int streams, int left_waves, int right_waves) {
  using P = JoinStep::Phase;
  std::vector<JoinStep> s;
  auto add = [&](P ph, int stream, int wave) { s.push_back(JoinStep{ph, stream, wave}); };
  const bool blocking = variant == kJoinBlocking || variant == kJoinBlockingOpt;
  if (blocking) {
    // one stream, whole tables: build side concat -> partition -> sizes -> shuffle -> build, then
    // the probe side likewise -> probe
    const P order[] = {P::ConcatLeft, P::PartitionLeft,  P::SizesLeft,  P::ShuffleLeft,  P::Build, P::ConcatRight,
                       P::PartitionRight, P::SizesRight, P::ShuffleRight, P::Probe, P::Drain};
    for (P ph : order) add(ph, 0, ph == P::Build || ph == P::Drain ? -1 : 0);
    return s;
  }
  const int k = std::max(1, streams);
  const int build_stream = k;  // the dedicated build stream
  for (int w = 0; w < left_waves; ++w)
    for (P ph : {P::PartitionLeft, P::SizesLeft, P::ShuffleLeft}) add(ph, w % k, w);
  if (variant == kJoinChunking) {
    add(P::Build, build_stream, -1);
    for (int w = 0; w < right_waves; ++w)
      for (P ph : {P::PartitionRight, P::SizesRight, P::ShuffleRight, P::Probe}) add(ph, w % k, w);
  } else {  // deferred synchronisation
    for (int w = 0; w < right_waves; ++w) {
      if (w >= k) add(P::Probe, (w - k) % k, w - k);  // the wave k back on this stream
      for (P ph : {P::PartitionRight, P::SizesRight, P::ShuffleRight}) add(ph, w % k, w);
      if (w == 0) add(P::Build, build_stream, -1);  // after the first probe-side shuffle is in flight
    }
    if (right_waves == 0) add(P::Build, build_stream, -1);
    for (int w = std::max(0, right_waves - k); w < right_waves; ++w) add(P::Probe, w % k, w);
  }
  add(P::Drain, 0, -1);
  return s;
}

namespace {

using Clock = std::chrono::steady_clock;

/// Columnar device rows (all int64 words).
struct Cols {
  std::vector<void*> col;
  uint64_t rows = 0;
};

class JoinRun {
 public:
  JoinRun(Ctx& ctx, const JoinSpecC& spec, const HostTable& build, const HostTable& probe, bool collect)
      : ctx_(ctx), spec_(spec), build_(build), probe_(probe), collect_(collect) {
    pool_.init(ctx.device, 0);
  }
  ~JoinRun();
  JoinOutcome run();

 private:
  struct Wave {
    const HostTable* src = nullptr;
    uint64_t row0 = 0, rows = 0;  // slice of this node's table
    void* slab = nullptr;         // destination-major columnar send slab
    std::vector<uint64_t> dest_cnt;
    std::vector<uint64_t> recv_cnt;
    void* recv = nullptr;         // per-source columnar receive blocks
    uint64_t recv_rows = 0;
    cudaEvent_t shuffled = nullptr;
  };
  struct Side {
    const HostTable* table = nullptr;
    std::vector<Wave> waves;
    int ncols = 0;
  };

  void* dalloc(size_t bytes, cudaStream_t s);
  void dfree(void* p, cudaStream_t s);
  cudaStream_t stream(int i) { return streams_.at(static_cast<size_t>(i)); }
  void wait(cudaStream_t s) {
    PSG_CUDA(cudaStreamSynchronize(s));
    ++host_syncs_;
  }
  void concat(Side& side, cudaStream_t s);
  void partition(Side& side, int w, cudaStream_t s);
  void sizes(Side& side, int w, cudaStream_t s);
  void shuffle(Side& side, int w, cudaStream_t s);
  void build(cudaStream_t s);
  void probe(int w, cudaStream_t s);

  Ctx& ctx_;
  // a pool of this run's own: its blocks are keyed by this run's streams, so it is emptied before
  // the streams are destroyed (the context pool would keep stale stream keys)
  DevicePool pool_;
  JoinSpecC spec_;
  const HostTable& build_;
  const HostTable& probe_;
  bool collect_;
  int n_ = 1, me_ = 0;
  std::vector<cudaStream_t> streams_;
  Side left_, right_;
  std::vector<void*> pinned_;
  // build
  DevBuf tkeys_, tcnt_, tstart_;
  std::vector<DevBuf> tpay_;
  LocalTableDev table_{};
  cudaEvent_t built_ = nullptr;
  // results
  uint64_t result_rows_ = 0, bytes_received_ = 0, host_syncs_ = 0;
  std::vector<std::vector<uint64_t>> out_cols_;  // collected result columns (host)
  std::vector<std::pair<void*, cudaStream_t>> raw_;  // per-allocation mode buffers still live
};

JoinRun::~JoinRun() {
  for (auto s : streams_) cudaStreamSynchronize(s);
  cudaStreamSynchronize(ctx_.comm);
  for (auto& [p, s] : raw_) cudaFree(p);
  tkeys_.reset();
  tcnt_.reset();
  tstart_.reset();
  tpay_.clear();
  pool_.release_cache();
  for (auto& side : {&left_, &right_})
    for (auto& w : side->waves)
      if (w.shuffled) cudaEventDestroy(w.shuffled);
  if (built_) cudaEventDestroy(built_);
  for (auto s : streams_) cudaStreamDestroy(s);
}

/// Blocking (the reference's PoolMode::PerAllocation): a synchronous cudaMalloc per buffer;
/// every other variant takes buffers from the engine's stream-ordered caching pool.
void* JoinRun::dalloc(size_t bytes, cudaStream_t s) {
  bytes = std::max<size_t>(bytes, 16);
  if (spec_.variant == kJoinBlocking) {
    void* p = nullptr;
    PSG_CUDA(cudaMalloc(&p, bytes));
    raw_.push_back({p, s});
    return p;
  }
  return pool_.alloc(bytes, s);
}
void JoinRun::dfree(void* p, cudaStream_t s) {
  if (!p) return;
  if (spec_.variant == kJoinBlocking) {
    PSG_CUDA(cudaStreamSynchronize(s));
    PSG_CUDA(cudaFree(p));
    raw_.erase(std::remove_if(raw_.begin(), raw_.end(), [&](const auto& x) { return x.first == p; }), raw_.end());
    return;
  }
  pool_.free(p, s);
}

/// Blocking variants: the node's whole table becomes one wave (concat of its chunks).
void JoinRun::concat(Side& side, cudaStream_t s) {
  uint64_t rows = 0;
  for (auto& w : side.waves) rows += w.rows;
  Wave all;
  all.src = side.table;
  all.row0 = side.waves.empty() ? 0 : side.waves.front().row0;
  all.rows = rows;
  side.waves.assign(1, all);
  wait(s);  // data-dependent (the reference's concat blocks its issuer)
}

/// H2D of the wave's rows, then destination histogram + scatter into the send slab.
void JoinRun::partition(Side& side, int wi, cudaStream_t s) {
  Wave& w = side.waves.at(static_cast<size_t>(wi));
  const int nc = side.ncols;
  const uint64_t n = w.rows;
  std::vector<void*> in(nc, nullptr);
  for (int c = 0; c < nc; ++c) {
    in[c] = dalloc(n * 8 + 16, s);
    if (n)
      PSG_CUDA(cudaMemcpyAsync(in[c], side.table->cols[c].data() + w.row0, n * 8, cudaMemcpyHostToDevice, s));
  }
  void* cnt = dalloc(n_ * 8, s);
  void* base = dalloc(n_ * 8, s);
  void* cursor = dalloc(n_ * 8, s);
  PSG_CUDA(cudaMemsetAsync(cnt, 0, n_ * 8, s));
  PSG_CUDA(cudaMemsetAsync(cursor, 0, n_ * 8, s));
  launch_part_hist(static_cast<const uint64_t*>(in[0]), n, n_, static_cast<unsigned long long*>(cnt), s);
  const size_t tb = exclusive_scan_u64(nullptr, nullptr, n_, nullptr, 0, s);
  void* tmp = dalloc(tb, s);
  exclusive_scan_u64(static_cast<unsigned long long*>(cnt), static_cast<unsigned long long*>(base), n_, tmp, tb, s);
  w.slab = dalloc(n * nc * 8 + 16, s);
  std::vector<const uint64_t*> inc(nc);
  for (int c = 0; c < nc; ++c) inc[c] = static_cast<const uint64_t*>(in[c]);
  if (n)
    launch_part_scatter(inc.data(), nc, n, 0, n_, static_cast<unsigned long long*>(base), static_cast<unsigned long long*>(cnt),
                        static_cast<unsigned long long*>(cursor), static_cast<uint64_t*>(w.slab), s);
  w.dest_cnt.assign(n_, 0);
  PSG_CUDA(cudaMemcpyAsync(w.dest_cnt.data(), cnt, n_ * 8, cudaMemcpyDeviceToHost, s));
  wait(s);  // data-dependent
  for (auto p : in) dfree(p, s);
  for (auto p : {cnt, base, cursor, tmp}) dfree(p, s);
}

/// All-to-all of the per-destination row counts (Fabric::all_to_all_sizes, net.hpp:105-118) over
/// NCCL on the communication stream; the host needs them to size the receive buffers.
void JoinRun::sizes(Side& side, int wi, cudaStream_t s) {
  Wave& w = side.waves.at(static_cast<size_t>(wi));
  std::vector<uint64_t> m(static_cast<size_t>(n_) * n_, 0);
  if (n_ == 1) {
    m[0] = w.dest_cnt[0];
  } else {
    cudaEvent_t e;
    PSG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    PSG_CUDA(cudaEventRecord(e, s));
    PSG_CUDA(cudaStreamWaitEvent(ctx_.comm, e, 0));
    cudaEventDestroy(e);
    void* d = dalloc(m.size() * 8, ctx_.comm);
    void* mine = dalloc(n_ * 8, ctx_.comm);
    PSG_CUDA(cudaMemcpyAsync(mine, w.dest_cnt.data(), n_ * 8, cudaMemcpyHostToDevice, ctx_.comm));
    PSG_NCCL_J(ncclAllGather(mine, d, n_, ncclUint64, ctx_.nccl, ctx_.comm));
    PSG_CUDA(cudaMemcpyAsync(m.data(), d, m.size() * 8, cudaMemcpyDeviceToHost, ctx_.comm));
    wait(ctx_.comm);  // data-dependent
    dfree(d, ctx_.comm);
    dfree(mine, ctx_.comm);
  }
  const ExchangePlan x = plan_exchange(m.data(), n_, me_);
  w.recv_cnt = x.recv_cnt;
  w.recv_rows = x.recv_rows;
}

/// Asynchronous shuffle of the wave's slab: grouped ncclSend/ncclRecv on the communication stream
/// after the partition; `shuffled` orders the consumers (build, probe) behind it.
void JoinRun::shuffle(Side& side, int wi, cudaStream_t s) {
  Wave& w = side.waves.at(static_cast<size_t>(wi));
  const int nc = side.ncols;
  PSG_CUDA(cudaEventCreateWithFlags(&w.shuffled, cudaEventDisableTiming));
  if (n_ == 1) {  // nothing leaves the GPU: the slab is the received block
    w.recv = w.slab;
    w.slab = nullptr;
    PSG_CUDA(cudaEventRecord(w.shuffled, s));
    return;
  }
  cudaEvent_t e;
  PSG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  PSG_CUDA(cudaEventRecord(e, s));
  PSG_CUDA(cudaStreamWaitEvent(ctx_.comm, e, 0));
  cudaEventDestroy(e);
  w.recv = dalloc(w.recv_rows * nc * 8 + 16, ctx_.comm);
  uint64_t soff = 0, roff = 0;
  PSG_NCCL_J(ncclGroupStart());
  for (int p = 0; p < n_; ++p) {
    const uint64_t sc = w.dest_cnt[p], rc = w.recv_cnt[p];
    if (sc) PSG_NCCL_J(ncclSend(static_cast<uint64_t*>(w.slab) + soff * nc, sc * nc, ncclUint64, p, ctx_.nccl, ctx_.comm));
    if (rc) PSG_NCCL_J(ncclRecv(static_cast<uint64_t*>(w.recv) + roff * nc, rc * nc, ncclUint64, p, ctx_.nccl, ctx_.comm));
    if (p != me_) bytes_received_ += rc * nc * 8;
    soff += sc;
    roff += rc;
  }
  PSG_NCCL_J(ncclGroupEnd());
  PSG_CUDA(cudaEventRecord(w.shuffled, ctx_.comm));
  dfree(w.slab, ctx_.comm);
  w.slab = nullptr;
}

/// Columns of a received block from source p: rows [off, off + cnt) of the per-source columnar
/// layout (column c of source p at recv + off * nc + c * cnt).
std::vector<const uint64_t*> block_cols(void* recv, uint64_t off, uint64_t cnt, int nc) {
  std::vector<const uint64_t*> cols(nc);
  for (int c = 0; c < nc; ++c) cols[c] = static_cast<const uint64_t*>(recv) + off * nc + c * cnt;
  return cols;
}

/// CSR hash table over every received build row (HashTable::build, ops.cpp:105-159: duplicates
/// kept); waits for all build-side shuffles.
void JoinRun::build(cudaStream_t s) {
  const int nc = left_.ncols;
  uint64_t n = 0;
  for (auto& w : left_.waves) {
    if (w.shuffled) PSG_CUDA(cudaStreamWaitEvent(s, w.shuffled, 0));
    n += w.recv_rows;
  }
  // gather the received blocks into one columnar image
  std::vector<DevBuf> all;
  for (int c = 0; c < nc; ++c) all.emplace_back(pool_, std::max<uint64_t>(n, 1) * 8, s);
  uint64_t at = 0;
  for (auto& w : left_.waves) {
    uint64_t off = 0;
    for (int p = 0; p < n_; ++p) {
      const uint64_t rc = w.recv_cnt.empty() ? 0 : w.recv_cnt[p];
      if (rc) {
        auto cols = block_cols(w.recv, off, rc, nc);
        for (int c = 0; c < nc; ++c)
          PSG_CUDA(cudaMemcpyAsync(all[c].as<uint64_t>() + at, cols[c], rc * 8, cudaMemcpyDeviceToDevice, s));
      }
      off += rc;
      at += rc;
    }
    dfree(w.recv, s);
    w.recv = nullptr;
  }
  uint64_t cap = 16;
  while (cap < 2 * n) cap <<= 1;
  int shift = 64;
  for (uint64_t c = cap; c > 1; c >>= 1) --shift;
  tkeys_ = DevBuf(pool_, cap * 8, s);
  tcnt_ = DevBuf(pool_, (cap + 1) * 4, s);
  tstart_ = DevBuf(pool_, (cap + 1) * 4, s);
  DevBuf cursor(pool_, (cap + 1) * 4, s), maxc(pool_, 4, s);
  PSG_CUDA(cudaMemsetAsync(maxc.p, 0, 4, s));
  PSG_CUDA(cudaMemsetAsync(cursor.p, 0, (cap + 1) * 4, s));
  launch_local_init(tkeys_.as<uint64_t>(), tcnt_.as<uint32_t>(), cap, s);
  launch_local_count(tkeys_.as<uint64_t>(), tcnt_.as<uint32_t>(), cap - 1, shift, all[0].as<uint64_t>(), n,
                     maxc.as<unsigned>(), s);
  const size_t tb = exclusive_scan_u32(nullptr, nullptr, cap + 1, nullptr, 0, s);
  DevBuf tmp(pool_, tb, s);
  exclusive_scan_u32(tcnt_.as<uint32_t>(), tstart_.as<uint32_t>(), cap + 1, tmp.p, tb, s);
  std::vector<const uint64_t*> src;
  std::vector<uint64_t*> dst;
  for (int c = 1; c < nc; ++c) {
    tpay_.emplace_back(pool_, std::max<uint64_t>(n, 1) * 8, s);
    src.push_back(all[c].as<uint64_t>());
    dst.push_back(tpay_.back().as<uint64_t>());
  }
  launch_local_fill(tkeys_.as<uint64_t>(), tstart_.as<uint32_t>(), cursor.as<uint32_t>(), cap - 1, shift, all[0].as<uint64_t>(),
                    src.data(), dst.data(), nc - 1, n, s);
  std::memset(&table_, 0, sizeof table_);
  table_.keys = tkeys_.as<uint64_t>();
  table_.cnt = tcnt_.as<uint32_t>();
  table_.start = tstart_.as<uint32_t>();
  table_.mask = cap - 1;
  table_.shift = shift;
  table_.npayload = nc - 1;
  for (int c = 0; c < nc - 1; ++c) table_.payload[c] = tpay_[c].as<uint64_t>();
  PSG_CUDA(cudaEventCreateWithFlags(&built_, cudaEventDisableTiming));
  PSG_CUDA(cudaEventRecord(built_, s));
  wait(s);  // data-dependent
}

/// Expanding probe of one received probe-side wave: every build match of every row, output
/// columns = build payload ++ probe columns (ops.cpp:193-200).
void JoinRun::probe(int wi, cudaStream_t s) {
  Wave& w = right_.waves.at(static_cast<size_t>(wi));
  const int nc = right_.ncols, np = table_.npayload;
  if (built_) PSG_CUDA(cudaStreamWaitEvent(s, built_, 0));
  if (w.shuffled) PSG_CUDA(cudaStreamWaitEvent(s, w.shuffled, 0));
  uint64_t off = 0;
  for (int p = 0; p < n_; ++p) {
    const uint64_t rc = w.recv_cnt.empty() ? 0 : w.recv_cnt[p];
    if (!rc) continue;
    auto cols = block_cols(w.recv, off, rc, nc);
    off += rc;
    void* counts = dalloc((rc + 1) * 4, s);
    void* offs = dalloc((rc + 1) * 4, s);
    PSG_CUDA(cudaMemsetAsync(counts, 0, (rc + 1) * 4, s));
    launch_expand_count(table_, cols[0], rc, static_cast<uint32_t*>(counts), s);
    const size_t tb = exclusive_scan_u32(nullptr, nullptr, rc + 1, nullptr, 0, s);
    void* tmp = dalloc(tb, s);
    exclusive_scan_u32(static_cast<uint32_t*>(counts), static_cast<uint32_t*>(offs), rc + 1, tmp, tb, s);
    uint32_t total = 0;
    PSG_CUDA(cudaMemcpyAsync(&total, static_cast<uint32_t*>(offs) + rc, 4, cudaMemcpyDeviceToHost, s));
    wait(s);  // data-dependent: the output size
    std::vector<void*> out(np + nc);
    std::vector<uint64_t*> outp(np + nc);
    for (int c = 0; c < np + nc; ++c) {
      out[c] = dalloc(std::max<uint64_t>(total, 1) * 8, s);
      outp[c] = static_cast<uint64_t*>(out[c]);
    }
    launch_expand_write(table_, cols[0], rc, static_cast<uint32_t*>(offs), cols.data(), nc, outp.data(), s);
    if (collect_ && total) {
      if (out_cols_.empty()) out_cols_.resize(np + nc);
      for (int c = 0; c < np + nc; ++c) {
        const size_t at = out_cols_[c].size();
        out_cols_[c].resize(at + total);
        PSG_CUDA(cudaMemcpyAsync(out_cols_[c].data() + at, out[c], total * 8ull, cudaMemcpyDeviceToHost, s));
      }
      wait(s);
    }
    result_rows_ += total;
    for (auto x : out) dfree(x, s);
    for (auto x : {counts, offs, tmp}) dfree(x, s);
  }
  dfree(w.recv, s);
  w.recv = nullptr;
  wait(s);  // data-dependent (the probe's output is handed to the sink)
}

JoinOutcome JoinRun::run() {
  n_ = ctx_.nranks;
  me_ = ctx_.rank;
  if (spec_.chunk_rows < 1) throw InvalidInput("chunk_rows must be >= 1");
  if (spec_.stream_count < 1) throw InvalidInput("stream_count must be >= 1");
  if (spec_.variant < 0 || spec_.variant > kJoinDeferred) throw InvalidInput("unknown join variant");
  if (n_ > 1 && ctx_.nccl == nullptr) throw InvalidInput("nranks > 1 needs psg_ctx_init_comm first");
  const bool blocking = spec_.variant == kJoinBlocking || spec_.variant == kJoinBlockingOpt;
  const int k = blocking ? 1 : spec_.stream_count;
  left_.table = &build_;
  right_.table = &probe_;
  left_.ncols = static_cast<int>(build_.cols.size());
  right_.ncols = static_cast<int>(probe_.cols.size());
  if (left_.ncols < 1 || right_.ncols < 1 || left_.ncols + right_.ncols > kMaxOut + 1)
    throw InvalidInput("join tables need a key column and at most kMaxOut columns");
  // chunk_rows waves (chunk_rows_split: at least one, possibly empty, chunk per side)
  for (Side* side : {&left_, &right_}) {
    const uint64_t rows = side->table->rows();
    for (uint64_t lo = 0; lo < rows; lo += spec_.chunk_rows) {
      Wave w;
      w.row0 = lo;
      w.rows = std::min<uint64_t>(spec_.chunk_rows, rows - lo);
      side->waves.push_back(w);
    }
    if (side->waves.empty()) side->waves.push_back(Wave{});
  }
  for (int i = 0; i <= k; ++i) {  // + the dedicated build stream
    cudaStream_t s;
    PSG_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    streams_.push_back(s);
  }
  const auto t0 = Clock::now();
  cudaEvent_t ev0, ev1;
  PSG_CUDA(cudaEventCreate(&ev0));
  PSG_CUDA(cudaEventCreate(&ev1));
  PSG_CUDA(cudaEventRecord(ev0, streams_[0]));
  int lw = static_cast<int>(left_.waves.size()), rw = static_cast<int>(right_.waves.size());
  if (!blocking && n_ > 1) {
    // wave agreement: ranks may hold different chunk counts; every rank issues the same collective
    // sequence, so waves pad to the maximum (empty waves still exchange sizes)
    uint64_t h[2] = {static_cast<uint64_t>(lw), static_cast<uint64_t>(rw)};
    DevBuf d(ctx_.pool, 16, ctx_.comm);
    PSG_CUDA(cudaMemcpyAsync(d.p, h, 16, cudaMemcpyHostToDevice, ctx_.comm));
    PSG_NCCL_J(ncclAllReduce(d.p, d.p, 2, ncclUint64, ncclMax, ctx_.nccl, ctx_.comm));
    PSG_CUDA(cudaMemcpyAsync(h, d.p, 16, cudaMemcpyDeviceToHost, ctx_.comm));
    wait(ctx_.comm);
    lw = static_cast<int>(h[0]);
    rw = static_cast<int>(h[1]);
    while (static_cast<int>(left_.waves.size()) < lw) left_.waves.push_back(Wave{});
    while (static_cast<int>(right_.waves.size()) < rw) right_.waves.push_back(Wave{});
  }
  using P = JoinStep::Phase;
  const auto steps = join_schedule(spec_.variant, k, lw, rw);
  for (const JoinStep& st : steps) {
    switch (st.phase) {
      case P::ConcatLeft: concat(left_, stream(st.stream)); break;
      case P::ConcatRight: concat(right_, stream(st.stream)); break;
      case P::PartitionLeft: partition(left_, st.wave, stream(st.stream)); break;
      case P::PartitionRight: partition(right_, st.wave, stream(st.stream)); break;
      case P::SizesLeft: sizes(left_, st.wave, stream(st.stream)); break;
      case P::SizesRight: sizes(right_, st.wave, stream(st.stream)); break;
      case P::ShuffleLeft: shuffle(left_, st.wave, stream(st.stream)); break;
      case P::ShuffleRight: shuffle(right_, st.wave, stream(st.stream)); break;
      case P::Build: build(stream(st.stream)); break;
      case P::Probe: probe(st.wave, stream(st.stream)); break;
      case P::Drain: break;
    }
  }
  for (auto s : streams_) PSG_CUDA(cudaStreamSynchronize(s));
  PSG_CUDA(cudaStreamSynchronize(ctx_.comm));
  PSG_CUDA(cudaEventRecord(ev1, streams_[0]));
  PSG_CUDA(cudaEventSynchronize(ev1));
  float ms = 0;
  PSG_CUDA(cudaEventElapsedTime(&ms, ev0, ev1));
  cudaEventDestroy(ev0);
  cudaEventDestroy(ev1);
  JoinOutcome o;
  o.runtime_s = std::chrono::duration<double>(Clock::now() - t0).count();
  o.device_ms = ms;
  o.result_rows = result_rows_;
  o.bytes_received = bytes_received_;
  o.left_waves = static_cast<uint64_t>(lw);
  o.right_waves = static_cast<uint64_t>(rw);
  o.host_syncs = host_syncs_;
  o.cols = std::move(out_cols_);
  return o;
}

}  // namespace

JoinOutcome run_join(Ctx& ctx, const JoinSpecC& spec, const HostTable& build, const HostTable& probe, bool collect) {
  PSG_CUDA(cudaSetDevice(ctx.device));
  JoinRun r(ctx, spec, build, probe, collect);
  return r.run();
}

}  // namespace psg
