// extern "C" boundary (include/psg.h). Every call catches psg::Error / std::exception and turns
// it into a psg_status code + thread-local message, mirroring the reference's exception classes.
#include <execinfo.h>
#include <signal.h>
#include <unistd.h>

#include <cmath>
#include <mutex>
#include <tuple>
#include <cstdlib>
#include <cstring>

#include "engine.hpp"
#include "jit.hpp"
#include "shuffle_plan.hpp"

using namespace psg;

struct psg_ctx {
  Ctx c;
};
struct psg_result {
  ResultRows r;
};
struct psg_staged {
  Staged* s = nullptr;
};

namespace {
thread_local std::string g_err;

// PSG_SEGV_TRACE=1: print a native backtrace on SIGSEGV/SIGABRT (debugging on the GPU box).
void segv_handler(int sig) {
  void* frames[64];
  const int n = backtrace(frames, 64);
  const char msg[] = "psg: fatal signal, native backtrace:\n";
  (void)!write(2, msg, sizeof msg - 1);
  backtrace_symbols_fd(frames, n, 2);
  signal(sig, SIG_DFL);
  raise(sig);
}
void maybe_install_trace() {
  static bool done = false;
  if (done) return;
  done = true;
  const char* e = std::getenv("PSG_SEGV_TRACE");
  if (e && e[0] == '1') {
    signal(SIGSEGV, segv_handler);
    signal(SIGABRT, segv_handler);
  }
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return PSG_OK;
  } catch (const Error& e) {
    g_err = e.what();
    return e.code();
  } catch (const std::bad_alloc& e) {
    g_err = std::string("host allocation failed: ") + e.what();
    return PSG_ERR_MEMORY_EXCEEDED;
  } catch (const std::exception& e) {
    g_err = e.what();
    return PSG_ERR_INTERNAL;
  }
}

HostBatch to_host(const psg_batch* b) {
  if (!b) throw InvalidInput("null batch");
  HostBatch h;
  for (uint32_t c = 0; c < b->ncols; ++c) {
    if (b->types[c] > 1) throw InvalidInput("unknown logical type");
    h.schema.fields.push_back(Field{b->names[c], static_cast<LType>(b->types[c])});
    h.cols.emplace_back(b->cols[c], b->cols[c] + b->nrows);
  }
  return h;
}

psg_result* to_result(const HostBatch& h) {
  auto* r = new psg_result;
  r->r.schema = h.schema;
  const uint64_t n = h.rows();
  const size_t nc = h.schema.size();
  r->r.nrows = n;
  r->r.words.resize(n * nc);
  for (size_t c = 0; c < nc; ++c)
    for (uint64_t i = 0; i < n; ++i) r->r.words[i * nc + c] = h.cols[c][i];
  return r;
}

Predicate to_pred(const psg_atom* atoms, uint32_t n) {
  Predicate p;
  for (uint32_t i = 0; i < n; ++i) {
    Atom a;
    a.column = atoms[i].column;
    a.op = cmp_op_from_string(atoms[i].op);
    a.lit_is_float = atoms[i].literal_is_float != 0;
    a.lit_i = atoms[i].literal_i;
    a.lit_f = atoms[i].literal_f;
    p.push_back(a);
  }
  return p;
}
}  // namespace

extern "C" {

int psg_abi_version(void) { return PSG_ABI_VERSION; }

int psg_shuffle_plan(const uint64_t* matrix, int n, int me, uint64_t* send_off, uint64_t* recv_off,
                     uint64_t* send_rows, uint64_t* recv_rows) {
  return guarded([&] {
    if (!matrix) throw InvalidInput("null count matrix");
    const ExchangePlan x = plan_exchange(matrix, n, me);
    for (int p = 0; p < n; ++p) {
      if (send_off) send_off[p] = x.send_off[p];
      if (recv_off) recv_off[p] = x.recv_off[p];
    }
    if (send_rows) *send_rows = x.send_rows;
    if (recv_rows) *recv_rows = x.recv_rows;
  });
}

int psg_pack_plan(const int64_t* lo, const int64_t* hi, int ncols, int64_t* min, int* shift, uint64_t* mask, int* fits) {
  return guarded([&] {
    if (!lo || !hi || ncols < 1 || ncols > kMaxOut) throw InvalidInput("pack plan: bad columns");
    const PackLayout L = plan_pack(lo, hi, ncols);
    for (int k = 0; k < ncols; ++k) {
      if (min) min[k] = L.min[k];
      if (shift) shift[k] = L.shift[k];
      if (mask) mask[k] = L.mask[k];
    }
    if (fits) *fits = L.fits ? 1 : 0;
  });
}

int psg_partition_of(const int64_t* keys, uint64_t n, uint32_t nparts, uint32_t* out) {
  return guarded([&] {
    if ((!keys || !out) && n) throw InvalidInput("null argument");
    if (nparts == 0) throw InvalidInput("nparts must be > 0");
    for (uint64_t i = 0; i < n; ++i) out[i] = partition_of_host(static_cast<uint64_t>(keys[i]), nparts);
  });
}

int psg_join_schedule(int variant, int stream_count, int left_waves, int right_waves, int32_t* out, size_t cap_steps,
                      size_t* nsteps) {
  return guarded([&] {
    if (variant < 0 || variant > kJoinDeferred) throw InvalidInput("unknown join variant");
    if (stream_count < 1 || left_waves < 0 || right_waves < 0) throw InvalidInput("bad schedule shape");
    const auto steps = join_schedule(variant, stream_count, left_waves, right_waves);
    if (nsteps) *nsteps = steps.size();
    for (size_t i = 0; i < steps.size() && i < cap_steps && out; ++i) {
      out[3 * i] = static_cast<int32_t>(steps[i].phase);
      out[3 * i + 1] = steps[i].stream;
      out[3 * i + 2] = steps[i].wave;
    }
  });
}

int psg_run_synthetic_join(psg_ctx* ctx, const psg_join_spec* spec, const psg_join_workload* workload, int collect_rows,
                           psg_join_stats* stats, psg_result** rows) {
  return guarded([&] {
    if (!ctx || !spec || !workload) throw InvalidInput("null argument");
    // the generated slice is kept for the next call with the same workload (benchmarks run every
    // variant over one generation; the tables are host inputs, like the reference harness's)
    static std::mutex mu;
    static std::tuple<uint64_t, uint64_t, int, double, uint64_t, int, int> last_key{};
    static HostTable build, probe;
    std::lock_guard<std::mutex> lk(mu);
    const auto key = std::make_tuple(workload->build_rows, workload->probe_rows, workload->payload_cols,
                                     workload->hit_ratio, workload->seed, ctx->c.rank, ctx->c.nranks);
    if (key != last_key || build.cols.empty()) {
      for (HostTable* t : {&build, &probe})
        for (auto& c : t->cols)
          if (!c.empty()) cudaHostUnregister(c.data());
      cudaGetLastError();
      build = HostTable{};
      probe = HostTable{};
      synthetic_join_tables(workload->seed, workload->build_rows, workload->probe_rows, workload->payload_cols,
                            workload->hit_ratio, ctx->c.rank, ctx->c.nranks, build, probe);
      // page-locked, like the pinned staging of the storage path: the waves' H2D copies run at
      // PCIe speed instead of through the driver's pageable bounce buffers
      for (HostTable* t : {&build, &probe})
        for (auto& c : t->cols)
          if (!c.empty() && cudaHostRegister(c.data(), c.size() * 8, cudaHostRegisterDefault) != cudaSuccess)
            cudaGetLastError();  // (stays pageable: slower copies, same results)
      last_key = key;
    }
    JoinSpecC js;
    js.variant = spec->variant;
    js.stream_count = spec->stream_count;
    js.chunk_rows = spec->chunk_rows;
    JoinOutcome o = run_join(ctx->c, js, build, probe, collect_rows != 0 && rows != nullptr);
    if (stats) {
      stats->runtime_s = o.runtime_s;
      stats->device_ms = o.device_ms;
      stats->result_rows = o.result_rows;
      stats->bytes_received = o.bytes_received;
      stats->left_waves = o.left_waves;
      stats->right_waves = o.right_waves;
      stats->host_syncs = o.host_syncs;
    }
    if (rows) {
      auto r = std::make_unique<psg_result>();
      // build payload ++ probe columns, "_p" on a name clash (ops.cpp:193-200)
      for (size_t c = 1; c < build.names.size(); ++c) r->r.schema.fields.push_back(Field{build.names[c], LType::Int64});
      for (const auto& nm : probe.names) {
        Field f{nm, LType::Int64};
        if (r->r.schema.index_of(f.name)) f.name += "_p";
        r->r.schema.fields.push_back(f);
      }
      const size_t nc = r->r.schema.size();
      const uint64_t n = o.cols.empty() ? 0 : o.cols[0].size();
      r->r.nrows = n;
      uint64_t* w = r->r.mutable_rows(n * nc);
      for (size_t c = 0; c < nc && !o.cols.empty(); ++c)
        for (uint64_t i = 0; i < n; ++i) w[i * nc + c] = o.cols[c][i];
      *rows = r.release();
    }
  });
}

int psg_plan_resolve(const char* plan_json, const char* data_root, int node, int nodes, char* out, size_t cap,
                     size_t* needed) {
  return guarded([&] {
    if (!plan_json || !data_root) throw InvalidInput("null plan or data root");
    const QueryPlan p = QueryPlan::from_json_text(plan_json, data_root, node, nodes);
    // {"scans":[{"table":..,"replicated":b,"paths":[..]}..],"shuffle":"id"|null}
    auto q = [](const std::string& x) {
      std::string o = "\"";
      for (char ch : x) {
        if (ch == '"' || ch == '\\') o += '\\';
        o += ch;
      }
      return o + "\"";
    };
    std::string j = "{\"scans\": [";
    for (size_t i = 0; i < p.scans.size(); ++i) {
      const ScanNode& sc = p.scans[i];
      j += (i ? ", " : "") + std::string("{\"table\": ") + q(sc.table) + ", \"replicated\": " +
           (sc.replicated ? "true" : "false") + ", \"paths\": [";
      for (size_t k = 0; k < sc.paths.size(); ++k) j += (k ? ", " : "") + q(sc.paths[k]);
      j += "]}";
    }
    const JoinNode* sj = p.shuffle_join();
    j += "], \"shuffle\": " + (sj ? q(sj->id) : std::string("null")) + "}";
    if (needed) *needed = j.size() + 1;
    if (out && cap) {
      const size_t n = std::min(cap - 1, j.size());
      std::memcpy(out, j.data(), n);
      out[n] = '\0';
    }
  });
}
const char* psg_last_error(void) { return g_err.c_str(); }

int psg_ctx_create(int device, int rank, int nranks, psg_ctx** out) {
  return guarded([&] {
    if (!out) throw InvalidInput("null out");
    maybe_install_trace();
    if (nranks < 1 || rank < 0 || rank >= nranks) throw InvalidInput("bad rank/nranks");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
      throw Error(PSG_ERR_CUDA, "no CUDA device visible: the B200 path has no CPU fallback");
    if (device < 0 || device >= ndev) throw InvalidInput("device ordinal out of range");
    auto ctx = std::make_unique<psg_ctx>();
    Ctx& c = ctx->c;
    c.device = device;
    c.rank = rank;
    c.nranks = nranks;
    PSG_CUDA(cudaSetDevice(device));
    cudaDeviceProp prop;
    PSG_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10) throw Error(PSG_ERR_CUDA, std::string("device is not sm_100-class: ") + prop.name);
    PSG_CUDA(cudaStreamCreateWithFlags(&c.compute, cudaStreamNonBlocking));
    PSG_CUDA(cudaStreamCreateWithFlags(&c.copy, cudaStreamNonBlocking));
    PSG_CUDA(cudaStreamCreateWithFlags(&c.comm, cudaStreamNonBlocking));
    PSG_CUDA(cudaEventCreate(&c.ev_a));
    PSG_CUDA(cudaEventCreate(&c.ev_b));
    c.pool.init(device, 0);
    // L2 fetch granularity: the late columns are gathered for a few percent of the rows, so a
    // miss should bring in the 32-byte sector it needs, not a wider line. PSG_L2_FETCH=<bytes>
    // (32..128; 0 = leave the driver default).
    static const long fetch = [] {
      const char* e = std::getenv("PSG_L2_FETCH");
      return e ? std::atol(e) : 32L;
    }();
    if (fetch > 0 && cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, static_cast<size_t>(fetch)) != cudaSuccess)
      cudaGetLastError();
    *out = ctx.release();
  });
}

int psg_comm_unique_id(void* out128) {
  return guarded([&] {
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) throw Error(PSG_ERR_NCCL, "ncclGetUniqueId failed");
    std::memcpy(out128, &id, sizeof id);
  });
}

int psg_ctx_init_comm(psg_ctx* ctx, const void* id128) {
  return guarded([&] {
    if (!ctx) throw InvalidInput("null ctx");
    PSG_CUDA(cudaSetDevice(ctx->c.device));
    if (ctx->c.nranks == 1) return;
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof id);
    const ncclResult_t r = ncclCommInitRank(&ctx->c.nccl, ctx->c.nranks, id, ctx->c.rank);
    if (r != ncclSuccess) throw Error(PSG_ERR_NCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));

  });
}

int psg_ctx_set_ingest(psg_ctx* ctx, int io_threads, uint64_t batch_bytes, int pinned_slots) {
  return guarded([&] {
    if (!ctx) throw InvalidInput("null ctx");
    if (io_threads >= 0) ctx->c.io_threads = io_threads;
    if (batch_bytes > 0) ctx->c.batch_bytes = batch_bytes;
    if (pinned_slots >= 0) ctx->c.pinned_slots = pinned_slots;
  });
}

int psg_ctx_set_semijoin(psg_ctx* ctx, int enabled) {
  return guarded([&] {
    if (!ctx) throw InvalidInput("null ctx");
    ctx->c.semijoin = enabled != 0;
  });
}

int psg_ctx_set_fused_shuffle(psg_ctx* ctx, int enabled) {
  return guarded([&] {
    if (!ctx) throw InvalidInput("null ctx");
    if (enabled && ctx->c.nranks > 1 && ctx->c.symm == nullptr) {
      // collective: every rank enables the fused path together (maps every peer's heap)
      const char* e = std::getenv("PSG_SYMM_MB");
      const size_t mb = e ? static_cast<size_t>(std::atoll(e)) : 4096;
      PSG_CUDA(cudaSetDevice(ctx->c.device));
      ctx->c.init_symmetric_heap(mb << 20);
    }
    if (enabled && ctx->c.nranks > 1 && ctx->c.symm_bytes == 0) throw InvalidInput("no symmetric heap (CUDA IPC unavailable)");
    ctx->c.p2p = enabled != 0 && ctx->c.symm_bytes > 0;
  });
}

void psg_ctx_destroy(psg_ctx* ctx) { delete ctx; }

int psg_execute_plan(psg_ctx* ctx, const char* plan_json, const char* data_root, int mode, psg_result** out) {
  return guarded([&] {
    if (!ctx || !plan_json || !data_root || !out) throw InvalidInput("null argument");
    if (ctx->c.io_threads == 0) {
      // default: plan.io_workers (resolved inside) -> use hardware threads when unset
      ctx->c.io_threads = 8;
    }
    auto r = std::make_unique<psg_result>();
    r->r = execute_plan(ctx->c, plan_json, data_root, mode, nullptr, true);
    *out = r.release();
  });
}

int psg_execute_local(psg_ctx* ctx, const char* plan_json, const char* data_root, int mode, psg_result** out) {
  return guarded([&] {
    if (!ctx || !plan_json || !data_root || !out) throw InvalidInput("null argument");
    if (ctx->c.io_threads == 0) ctx->c.io_threads = 8;
    auto r = std::make_unique<psg_result>();
    r->r = execute_local(ctx->c, plan_json, data_root, mode);
    *out = r.release();
  });
}

int psg_ingest_probe(psg_ctx* ctx, const char* plan_json, const char* data_root, psg_stats* out) {
  return guarded([&] {
    if (!ctx || !plan_json || !data_root || !out) throw InvalidInput("null argument");
    if (ctx->c.io_threads == 0) ctx->c.io_threads = 8;
    *out = ingest_only(ctx->c, plan_json, data_root).stats;
  });
}

int psg_stage_plan(psg_ctx* ctx, const char* plan_json, const char* data_root, psg_staged** out) {
  return guarded([&] {
    if (!ctx || !plan_json || !data_root || !out) throw InvalidInput("null argument");
    if (ctx->c.io_threads == 0) ctx->c.io_threads = 8;
    auto s = std::make_unique<psg_staged>();
    s->s = stage_plan(ctx->c, plan_json, data_root);
    *out = s.release();
  });
}

int psg_execute_staged(psg_ctx* ctx, psg_staged* staged, int mode, psg_result** out, psg_stats* stats) {
  return guarded([&] {
    if (!ctx || !staged) throw InvalidInput("null argument");
    auto r = std::make_unique<psg_result>();
    r->r = execute_plan(ctx->c, "", "", mode, staged->s, out != nullptr);
    if (stats) *stats = r->r.stats;
    if (out) *out = r.release();
  });
}

void psg_staged_free(psg_staged* s) {
  if (!s) return;
  free_staged(s->s);
  delete s;
}

int psg_result_shape(const psg_result* r, uint64_t* nrows, uint32_t* ncols) {
  return guarded([&] {
    if (!r) throw InvalidInput("null result");
    if (nrows) *nrows = r->r.nrows;
    if (ncols) *ncols = static_cast<uint32_t>(r->r.schema.size());
  });
}

int psg_result_field(const psg_result* r, uint32_t col, const char** name, int* type) {
  return guarded([&] {
    if (!r || col >= r->r.schema.size()) throw InvalidInput("column out of range");
    if (name) *name = r->r.schema.fields[col].name.c_str();
    if (type) *type = static_cast<int>(r->r.schema.fields[col].type);
  });
}

const uint64_t* psg_result_data(const psg_result* r) { return r ? r->r.data() : nullptr; }

int psg_result_stats(const psg_result* r, psg_stats* out) {
  return guarded([&] {
    if (!r || !out) throw InvalidInput("null argument");
    *out = r->r.stats;
  });
}

int psg_result_checksum(const psg_result* r, uint64_t* rowhash, uint64_t* colsums, uint32_t ncols_cap) {
  return guarded([&] {
    if (!r || !rowhash) throw InvalidInput("null argument");
    const uint64_t n = r->r.nrows;
    const size_t nc = r->r.schema.size();
    const uint64_t* w = r->r.data();
    // sum over rows of FNV-1a64 of the row's little-endian bytes (mod 2^64): order-independent and
    // additive over ranks, the reference harness's result checksum (hashing.hpp fnv1a64)
    uint64_t h = 0;
    std::vector<uint64_t> cs(nc, 0);
    for (uint64_t i = 0; i < n; ++i) {
      uint64_t f = 0xcbf29ce484222325ULL;
      for (size_t c = 0; c < nc; ++c) {
        const uint64_t x = w[i * nc + c];
        cs[c] += x;
        for (int b = 0; b < 8; ++b) f = (f ^ ((x >> (8 * b)) & 0xFF)) * 0x100000001b3ULL;
      }
      h += f;
    }
    *rowhash = h;
    if (colsums)
      for (size_t c = 0; c < nc && c < ncols_cap; ++c) colsums[c] = cs[c];
  });
}

void psg_result_free(psg_result* r) { delete r; }

int psg_filter(psg_ctx* ctx, const psg_batch* in, const psg_atom* atoms, uint32_t natoms, psg_result** out) {
  return guarded([&] {
    if (!ctx || !out) throw InvalidInput("null argument");
    HostBatch h = to_host(in);
    *out = to_result(op_filter(ctx->c, h, to_pred(atoms, natoms)));
  });
}

int psg_partition(psg_ctx* ctx, const psg_batch* in, const char* key_column, uint32_t nparts, int hash_kind,
                  psg_result** out, uint64_t* part_rows) {
  return guarded([&] {
    if (!ctx || !out || !key_column) throw InvalidInput("null argument");
    HostBatch h = to_host(in);
    std::vector<uint64_t> pr;
    *out = to_result(op_partition(ctx->c, h, key_column, nparts, hash_kind == 1, pr));
    if (part_rows) std::memcpy(part_rows, pr.data(), pr.size() * 8);
  });
}

int psg_codec_decompress(psg_ctx* ctx, int codec, uint64_t n, const void* const* src, const uint64_t* src_len,
                         void* const* dst, const uint64_t* dst_len) {
  return guarded([&] {
    if (!ctx || (n && (!src || !src_len || !dst || !dst_len))) throw InvalidInput("null argument");
    if (codec != 0 && codec != 1) throw InvalidInput("unknown codec");
    op_codec_decompress(ctx->c, codec, n, src, src_len, dst, dst_len);
  });
}

struct psg_hashtable {
  psg::GpuHashTable* t = nullptr;
  ~psg_hashtable() { psg::op_hashtable_free(t); }
};

int psg_hashtable_build(psg_ctx* ctx, const psg_batch* batches, uint32_t nbatches, const char* key_column, int hash_kind,
                        psg_hashtable** out) {
  return guarded([&] {
    if (!ctx || !out || !key_column || (nbatches && !batches)) throw InvalidInput("null argument");
    if (hash_kind != 0 && hash_kind != 1) throw InvalidInput("unknown hash kind");
    std::vector<HostBatch> hs;
    for (uint32_t i = 0; i < nbatches; ++i) hs.push_back(to_host(&batches[i]));
    auto h = std::make_unique<psg_hashtable>();
    h->t = op_hashtable_build(ctx->c, hs, key_column);
    *out = h.release();
  });
}

int psg_hashtable_shape(const psg_hashtable* t, uint64_t* rows, uint32_t* payload_cols) {
  return guarded([&] {
    if (!t) throw InvalidInput("null argument");
    const HostBatch& h = op_hashtable_host(*t->t);
    if (rows) *rows = h.rows();
    if (payload_cols) *payload_cols = static_cast<uint32_t>(h.schema.size() - 1);
  });
}

int psg_hashtable_row(const psg_hashtable* t, const char* key_column, uint64_t row, int64_t* key, uint64_t* payload) {
  return guarded([&] {
    if (!t || !key_column) throw InvalidInput("null argument");
    const HostBatch& h = op_hashtable_host(*t->t);
    if (row >= h.rows()) throw InvalidInput("row out of range");
    const size_t k = h.schema.require(key_column);
    if (key) *key = static_cast<int64_t>(h.cols[k][row]);
    size_t o = 0;
    for (size_t c = 0; c < h.cols.size(); ++c)
      if (c != k && payload) payload[o++] = h.cols[c][row];
  });
}

int psg_hashtable_lookup(psg_ctx* ctx, const psg_hashtable* t, const int64_t* keys, uint64_t n, uint64_t* offsets,
                         uint64_t* rows_out, uint64_t cap, uint64_t* total) {
  return guarded([&] {
    if (!ctx || !t || (n && !keys) || !offsets || !total) throw InvalidInput("null argument");
    std::vector<uint64_t> off;
    auto rows = op_hashtable_lookup(ctx->c, *t->t, std::vector<int64_t>(keys, keys + n), off);
    std::memcpy(offsets, off.data(), (n + 1) * 8);
    *total = rows.size();
    if (rows.size() > cap) throw InvalidInput("lookup result exceeds the output capacity");
    if (!rows.empty()) std::memcpy(rows_out, rows.data(), rows.size() * 8);
  });
}

int psg_hashtable_probe(psg_ctx* ctx, const psg_hashtable* t, const psg_batch* probe, const char* probe_key,
                        psg_result** out) {
  return guarded([&] {
    if (!ctx || !t || !probe_key || !out) throw InvalidInput("null argument");
    *out = to_result(op_hashtable_probe(ctx->c, *t->t, to_host(probe), probe_key));
  });
}

void psg_hashtable_free(psg_hashtable* t) { delete t; }

int psg_concat(psg_ctx* ctx, const psg_batch* batches, uint32_t nbatches, psg_result** out) {
  return guarded([&] {
    if (!ctx || !out || (nbatches && !batches)) throw InvalidInput("null argument");
    std::vector<HostBatch> hs;
    for (uint32_t i = 0; i < nbatches; ++i) hs.push_back(to_host(&batches[i]));
    *out = to_result(op_concat(ctx->c, hs));
  });
}

int psg_hash_join(psg_ctx* ctx, const psg_batch* build, const char* build_key, const psg_batch* probe,
                  const char* probe_key, psg_result** out) {
  return guarded([&] {
    if (!ctx || !out || !build_key || !probe_key) throw InvalidInput("null argument");
    *out = to_result(op_hash_join(ctx->c, to_host(build), build_key, to_host(probe), probe_key));
  });
}

int psg_psto_write(const char* path, const psg_batch* batch, uint64_t row_group_rows, int codec,
                   uint64_t* groups_written) {
  return guarded([&] {
    HostBatch h = to_host(batch);
    if (codec != 0 && codec != 1) throw InvalidInput("unknown codec");
    PstoWriter w(path, h.schema, row_group_rows, static_cast<Codec>(codec));
    std::vector<const uint64_t*> ptrs;
    for (auto& c : h.cols) ptrs.push_back(c.data());
    if (h.rows()) w.append(ptrs.data(), h.rows());
    TableMeta m = w.finish();
    if (groups_written) *groups_written = m.groups.size();
  });
}

int psg_psto_inspect(const char* path, uint64_t* rows, uint32_t* ncols, uint64_t* groups, int* codec) {
  return guarded([&] {
    TableMeta m = read_footer(path);
    if (rows) *rows = m.total_rows();
    if (ncols) *ncols = static_cast<uint32_t>(m.schema.size());
    if (groups) *groups = m.groups.size();
    if (codec) *codec = static_cast<int>(m.codec);
  });
}

int psg_gen_tpch(const char* out_dir, double scale, int nodes, int devices, uint64_t seed, int codec,
                 uint64_t row_group_bytes, int threads) {
  return guarded([&] {
    if (codec != 0 && codec != 1) throw InvalidInput("unknown codec");
    gen_tpch(out_dir, scale, nodes, devices, seed, static_cast<Codec>(codec), row_group_bytes, threads);
  });
}

int psg_gen_synthetic(const char* out_dir, int nodes, int devices, uint64_t seed, int codec, uint64_t row_group_bytes,
                      uint64_t build_rows, uint64_t probe_rows, int payload_cols, double hit_ratio) {
  return guarded([&] {
    if (!out_dir) throw InvalidInput("null argument");
    if (codec != 0 && codec != 1) throw InvalidInput("unknown codec");
    gen_synthetic(out_dir, nodes, devices, seed, static_cast<Codec>(codec), row_group_bytes, build_rows, probe_rows,
                  payload_cols, hit_ratio);
  });
}

int psg_jit_selftest(char* log, size_t cap) {
  std::string l;
  int f = 0;
  const int rc = guarded([&] { f = jit_selftest(l); });
  if (log && cap) {
    std::strncpy(log, l.c_str(), cap - 1);
    log[cap - 1] = '\0';
  }
  return rc != PSG_OK ? -1 : f;
}

double psg_tmin(uint64_t ssd_read_size_agg, double ssd_read_bw_agg, uint64_t net_recv_size_node, double net_bw) {
  // t_min (bench.cpp:35-40): invalid inputs return NaN (the C++ API throws InvalidInput).
  if (ssd_read_size_agg == 0 || ssd_read_bw_agg <= 0 || net_bw <= 0) {
    g_err = "invalid input: t_min inputs must be positive";
    return std::nan("");
  }
  const double storage = static_cast<double>(ssd_read_size_agg) / ssd_read_bw_agg;
  const double net = static_cast<double>(net_recv_size_node) / net_bw;
  return storage > net ? storage : net;
}

}  // extern "C"
