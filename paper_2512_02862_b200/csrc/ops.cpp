// Operator adapters (ops.hpp:35-83): host ChunkBatch -> HBM -> sm_100a kernel -> host.
// They exist so the reference's operator-level tests (core_ops_test.cpp) can run unchanged in
// spirit against the GPU kernels; the plan executor never goes through them.
#include <numeric>

#include "engine.hpp"
#include "jit.hpp"

namespace psg {

namespace {

struct Uploaded {
  std::vector<DevBuf> cols;
};

Uploaded upload(Ctx& ctx, const HostBatch& b) {
  Uploaded u;
  const uint64_t n = b.rows();
  for (auto& c : b.cols) {
    u.cols.emplace_back(ctx.pool, std::max<uint64_t>(n, 1) * 8 + 16, ctx.compute);
    if (n) PSG_CUDA(cudaMemcpyAsync(u.cols.back().p, c.data(), n * 8, cudaMemcpyHostToDevice, ctx.compute));
  }
  return u;
}

std::vector<uint64_t> download(Ctx& ctx, const DevBuf& d, uint64_t n) {
  std::vector<uint64_t> out(n);
  if (n) PSG_CUDA(cudaMemcpyAsync(out.data(), d.p, n * 8, cudaMemcpyDeviceToHost, ctx.compute));
  return out;
}

void check_batch(const HostBatch& b) {
  if (b.cols.size() != b.schema.size()) throw InvalidInput("batch column count does not match schema");
  for (auto& c : b.cols)
    if (c.size() != b.rows()) throw InvalidInput("ragged batch: column row counts differ");
  if (b.cols.size() > static_cast<size_t>(kMaxIn)) throw InvalidInput("too many columns for one batch");
}

}  // namespace

void op_codec_decompress(Ctx& ctx, int codec, uint64_t n, const void* const* src, const uint64_t* src_len,
                         void* const* dst, const uint64_t* dst_len) {
  PSG_CUDA(cudaSetDevice(ctx.device));
  if (codec == 0) {  // identity (codec_decompress returns the bytes as they are)
    for (uint64_t i = 0; i < n; ++i) {
      if (src_len[i] != dst_len[i]) throw IoFailure("inflate failed");
      if (src_len[i]) std::memcpy(dst[i], src[i], src_len[i]);
    }
    return;
  }
  // pack the streams 16-byte aligned into one upload, decode into one aligned output image
  uint64_t cbytes = 0, dbytes = 0;
  std::vector<uint64_t> coff(n), doff(n);
  for (uint64_t i = 0; i < n; ++i) {
    if (src_len[i] > 0xFFFFFFF0ull || dst_len[i] > 0xFFFFFFF0ull) throw InvalidInput("chunk larger than 4 GiB");
    coff[i] = cbytes;
    doff[i] = dbytes;
    cbytes += (src_len[i] + 15) & ~15ULL;
    dbytes += (dst_len[i] + 15) & ~15ULL;
  }
  if (n == 0) return;
  std::vector<uint8_t> host(cbytes + 16, 0);
  for (uint64_t i = 0; i < n; ++i)
    if (src_len[i]) std::memcpy(host.data() + coff[i], src[i], src_len[i]);
  DevBuf cdev(ctx.pool, host.size(), ctx.compute), ddev(ctx.pool, dbytes + 16, ctx.compute),
      jdev(ctx.pool, n * sizeof(InflateJob), ctx.compute), err(ctx.pool, sizeof(unsigned int), ctx.compute);
  std::vector<InflateJob> jobs(n);
  for (uint64_t i = 0; i < n; ++i)
    jobs[i] = InflateJob{cdev.as<uint8_t>() + coff[i], ddev.as<uint8_t>() + doff[i], static_cast<uint32_t>(src_len[i]),
                         static_cast<uint32_t>(dst_len[i])};
  PSG_CUDA(cudaMemcpyAsync(cdev.p, host.data(), host.size(), cudaMemcpyHostToDevice, ctx.compute));
  PSG_CUDA(cudaMemcpyAsync(jdev.p, jobs.data(), n * sizeof(InflateJob), cudaMemcpyHostToDevice, ctx.compute));
  PSG_CUDA(cudaMemsetAsync(err.p, 0, sizeof(unsigned int), ctx.compute));
  launch_inflate(jdev.as<InflateJob>(), static_cast<uint32_t>(n), err.as<unsigned int>(), ctx.compute);
  unsigned int e = 0;
  PSG_CUDA(cudaMemcpyAsync(&e, err.p, sizeof e, cudaMemcpyDeviceToHost, ctx.compute));
  PSG_CUDA(cudaStreamSynchronize(ctx.compute));
  if (e) throw IoFailure("inflate failed");
  std::vector<uint8_t> out(dbytes);
  PSG_CUDA(cudaMemcpy(out.data(), ddev.p, dbytes, cudaMemcpyDeviceToHost));
  for (uint64_t i = 0; i < n; ++i)
    if (dst_len[i]) std::memcpy(dst[i], out.data() + doff[i], dst_len[i]);
}

HostBatch op_filter(Ctx& ctx, const HostBatch& in, const Predicate& pred) {
  PSG_CUDA(cudaSetDevice(ctx.device));
  check_batch(in);
  const uint64_t n = in.rows();
  const int nc = static_cast<int>(in.schema.size());
  // registers: predicate columns first (bound by name, BoundPredicate predicate.cpp:94-100)
  std::vector<int> reg_col;  // reg -> column
  std::vector<int> col_reg(nc, -1);
  for (auto& a : pred) {
    const int c = static_cast<int>(in.schema.require(a.column));
    if (col_reg[c] < 0) {
      col_reg[c] = static_cast<int>(reg_col.size());
      reg_col.push_back(c);
    }
  }
  const int npred = static_cast<int>(reg_col.size());
  for (int c = 0; c < nc; ++c)
    if (col_reg[c] < 0) {
      col_reg[c] = static_cast<int>(reg_col.size());
      reg_col.push_back(c);
    }
  if (pred.size() > static_cast<size_t>(kMaxAtoms)) throw InvalidInput("too many predicate atoms");
  HostBatch out;
  out.schema = in.schema;
  out.cols.resize(nc);
  if (n == 0) return out;
  Uploaded u = upload(ctx, in);
  Segment sg;
  std::memset(&sg, 0, sizeof sg);
  for (size_t r = 0; r < reg_col.size(); ++r) sg.col[r] = u.cols[reg_col[r]].as<uint64_t>();
  sg.rows = n;
  sg.tile_begin = 0;
  const uint64_t T = static_cast<uint64_t>(scan_tile_rows());
  const uint64_t ntiles = (n + T - 1) / T;
  DevBuf dseg(ctx.pool, sizeof(Segment), ctx.compute), dtile(ctx.pool, ntiles * 4, ctx.compute);
  PSG_CUDA(cudaMemcpyAsync(dseg.p, &sg, sizeof sg, cudaMemcpyHostToDevice, ctx.compute));
  PSG_CUDA(cudaMemsetAsync(dtile.p, 0, ntiles * 4, ctx.compute));  // single segment
  ScanProgram p;
  std::memset(&p, 0, sizeof p);
  p.n_in = nc;
  p.n_pred = npred;
  p.n_early = npred;
  p.n_regs = std::max(1, nc);
  p.n_atoms = static_cast<int>(pred.size());
  for (size_t a = 0; a < pred.size(); ++a) {
    const int c = static_cast<int>(in.schema.require(pred[a].column));
    AtomDesc& d = p.atoms[a];
    d.reg = col_reg[c];
    d.op = static_cast<int>(pred[a].op);
    d.is_float = in.schema.fields[c].type == LType::Float64;
    if (d.is_float) {
      const double v = pred[a].as_float();
      std::memcpy(&d.lit, &v, 8);
    } else {
      d.lit = static_cast<uint64_t>(pred[a].as_int());
    }
  }
  p.part_key_reg = -1;
  p.key_reg = -1;
  // pass 1: per-tile counts; exclusive scan -> tile offsets; pass 2: ordered compaction
  DevBuf counts(ctx.pool, (ntiles + 1) * 8, ctx.compute), offs(ctx.pool, (ntiles + 1) * 8, ctx.compute);
  PSG_CUDA(cudaMemsetAsync(counts.p, 0, (ntiles + 1) * 8, ctx.compute));
  ScanProgram pc = p;
  pc.sink = SINK_COUNT;
  pc.tile_counts = counts.as<unsigned long long>();
  fused_scan(pc, dseg.as<Segment>(), dtile.as<uint32_t>(), 1, ntiles, ctx.compute);
  size_t tb = exclusive_scan_u64(nullptr, nullptr, ntiles + 1, nullptr, 0, ctx.compute);
  DevBuf tmp(ctx.pool, tb, ctx.compute);
  exclusive_scan_u64(counts.as<unsigned long long>(), offs.as<unsigned long long>(), ntiles + 1, tmp.p, tb, ctx.compute);
  uint64_t total = 0;
  PSG_CUDA(cudaMemcpyAsync(&total, offs.as<uint64_t>() + ntiles, 8, cudaMemcpyDeviceToHost, ctx.compute));
  PSG_CUDA(cudaStreamSynchronize(ctx.compute));
  std::vector<DevBuf> oc;
  ScanProgram pm = p;
  pm.sink = SINK_MATERIALIZE;
  pm.n_out = nc;
  for (int c = 0; c < nc; ++c) {
    oc.emplace_back(ctx.pool, std::max<uint64_t>(total, 1) * 8, ctx.compute);
    pm.out_reg[c] = col_reg[c];
    pm.out_col[c] = oc.back().as<uint64_t>();
  }
  pm.out_cap = total;
  pm.tile_offsets = offs.as<uint64_t>();
  DevBuf cnt(ctx.pool, 8, ctx.compute);
  pm.out_count = cnt.as<unsigned long long>();
  fused_scan(pm, dseg.as<Segment>(), dtile.as<uint32_t>(), 1, ntiles, ctx.compute);
  for (int c = 0; c < nc; ++c) out.cols[c] = download(ctx, oc[c], total);
  PSG_CUDA(cudaStreamSynchronize(ctx.compute));
  return out;
}

HostBatch op_partition(Ctx& ctx, const HostBatch& in, const std::string& key, uint32_t nparts, int identity,
                       std::vector<uint64_t>& part_rows) {
  PSG_CUDA(cudaSetDevice(ctx.device));
  check_batch(in);
  if (nparts < 1) throw InvalidInput("node count must be >= 1");
  const size_t kc = in.schema.require(key);
  if (in.schema.fields[kc].type != LType::Int64) throw InvalidInput("partition key must be int64: " + key);
  const uint64_t n = in.rows();
  const int nc = static_cast<int>(in.schema.size());
  HostBatch out;
  out.schema = in.schema;
  out.cols.resize(nc);
  part_rows.assign(nparts, 0);
  if (n == 0) return out;
  if (n >= (1ull << 32)) throw InvalidInput("op-level partition supports < 2^32 rows");
  Uploaded u = upload(ctx, in);
  DevBuf ids(ctx.pool, n * 4, ctx.compute), ids2(ctx.pool, n * 4, ctx.compute);
  DevBuf idx(ctx.pool, n * 4, ctx.compute), idx2(ctx.pool, n * 4, ctx.compute);
  launch_part_ids(u.cols[kc].as<uint64_t>(), n, static_cast<int>(nparts), identity, ids.as<uint32_t>(), ctx.compute);
  launch_iota_u32(idx.as<uint32_t>(), n, ctx.compute);
  int bits = 1;
  while ((1u << bits) < nparts) ++bits;
  size_t tb = sort_pairs_u32(nullptr, nullptr, nullptr, nullptr, n, bits, nullptr, 0, ctx.compute);
  DevBuf tmp(ctx.pool, tb, ctx.compute);
  // stable LSD radix sort by partition id keeps input order within each partition
  sort_pairs_u32(ids.as<uint32_t>(), ids2.as<uint32_t>(), idx.as<uint32_t>(), idx2.as<uint32_t>(), n, bits, tmp.p, tb,
                 ctx.compute);
  std::vector<DevBuf> oc;
  std::vector<const uint64_t*> ip;
  std::vector<uint64_t*> op;
  for (int c = 0; c < nc; ++c) {
    oc.emplace_back(ctx.pool, n * 8, ctx.compute);
    ip.push_back(u.cols[c].as<uint64_t>());
    op.push_back(oc.back().as<uint64_t>());
  }
  launch_gather(ip.data(), nc, idx2.as<uint32_t>(), n, op.data(), ctx.compute);
  std::vector<uint32_t> sorted(n);
  PSG_CUDA(cudaMemcpyAsync(sorted.data(), ids2.p, n * 4, cudaMemcpyDeviceToHost, ctx.compute));
  for (int c = 0; c < nc; ++c) out.cols[c] = download(ctx, oc[c], n);
  PSG_CUDA(cudaStreamSynchronize(ctx.compute));
  for (uint32_t d : sorted) part_rows[d]++;
  return out;
}

// ------------------------------------------------------------------ HashTable (ops.hpp:49-82)
/// GPU analog of the reference's chained HashTable (ops.cpp:105-222): the build batches are
/// concatenated in HBM (the "materialised build side", row r = r-th row of the concatenation),
/// and an open-addressing CSR index maps each key to the build-row indices that carry it
/// (duplicates keep every row). lookup returns those indices; probe expands every probe row by
/// its matches and gathers the build payload.
struct GpuHashTable {
  Ctx* ctx = nullptr;
  Schema schema;          // build schema
  size_t key = 0;         // key column index
  Schema payload_schema;  // build schema minus the key
  uint64_t rows = 0, cap = 0;
  int shift = 64;
  std::vector<DevBuf> cols;  // materialised build side (all columns), HBM
  DevBuf keys, cnt, start, rowidx;
  LocalTableDev dev{};
  HostBatch host;  // the same rows on the host (key_at / payload_at)
};

namespace {

HostBatch concat_host(const std::vector<HostBatch>& batches) {
  if (batches.empty()) throw InvalidInput("concat needs at least one batch");
  HostBatch out;
  out.schema = batches[0].schema;
  out.cols.resize(out.schema.size());
  for (const auto& b : batches) {
    check_batch(b);
    if (b.schema.size() != out.schema.size()) throw InvalidInput("concat: batches have different schemas");
    for (size_t c = 0; c < b.schema.size(); ++c)
      if (b.schema.fields[c].name != out.schema.fields[c].name || b.schema.fields[c].type != out.schema.fields[c].type)
        throw InvalidInput("concat: batches have different schemas");
    for (size_t c = 0; c < b.cols.size(); ++c) out.cols[c].insert(out.cols[c].end(), b.cols[c].begin(), b.cols[c].end());
  }
  return out;
}

/// Expanding join of `probe_keys` (device, n rows) against t: per key the matching build-row
/// indices, CSR (offsets on the device, n + 1 entries; returns the total match count).
uint64_t expand_rows(Ctx& ctx, const GpuHashTable& t, const uint64_t* probe_keys, uint64_t n, DevBuf& offs,
                     DevBuf& rows_out) {
  DevBuf counts(ctx.pool, (n + 1) * 4, ctx.compute);
  offs = DevBuf(ctx.pool, (n + 1) * 4, ctx.compute);
  PSG_CUDA(cudaMemsetAsync(counts.p, 0, (n + 1) * 4, ctx.compute));
  if (n) launch_expand_count(t.dev, probe_keys, n, counts.as<uint32_t>(), ctx.compute);
  const size_t tb = exclusive_scan_u32(nullptr, nullptr, n + 1, nullptr, 0, ctx.compute);
  DevBuf tmp(ctx.pool, std::max<size_t>(tb, 8), ctx.compute);
  exclusive_scan_u32(counts.as<uint32_t>(), offs.as<uint32_t>(), n + 1, tmp.p, tb, ctx.compute);
  uint32_t total = 0;
  PSG_CUDA(cudaMemcpyAsync(&total, offs.as<uint32_t>() + n, 4, cudaMemcpyDeviceToHost, ctx.compute));
  PSG_CUDA(cudaStreamSynchronize(ctx.compute));
  rows_out = DevBuf(ctx.pool, std::max<uint64_t>(total, 1) * 8, ctx.compute);
  uint64_t* outp = rows_out.as<uint64_t>();
  if (total) launch_expand_write(t.dev, probe_keys, n, offs.as<uint32_t>(), nullptr, 0, &outp, ctx.compute);
  return total;
}

}  // namespace

GpuHashTable* op_hashtable_build(Ctx& ctx, const std::vector<HostBatch>& batches, const std::string& key_column) {
  PSG_CUDA(cudaSetDevice(ctx.device));
  auto t = std::make_unique<GpuHashTable>();
  t->ctx = &ctx;
  t->host = concat_host(batches);
  t->schema = t->host.schema;
  t->key = t->schema.require(key_column);
  if (t->schema.fields[t->key].type != LType::Int64) throw InvalidInput("join key must be int64: " + key_column);
  for (size_t c = 0; c < t->schema.size(); ++c)
    if (c != t->key) t->payload_schema.fields.push_back(t->schema.fields[c]);
  const uint64_t nb = t->rows = t->host.rows();
  if (nb >= (1ULL << 32)) throw InvalidInput("hash table build side exceeds 2^32 rows");
  Uploaded u = upload(ctx, t->host);
  t->cols = std::move(u.cols);
  t->cap = 16;
  while (t->cap < 2 * nb) t->cap <<= 1;
  t->shift = 64;
  for (uint64_t c = t->cap; c > 1; c >>= 1) --t->shift;
  t->keys = DevBuf(ctx.pool, t->cap * 8, ctx.compute);
  t->cnt = DevBuf(ctx.pool, (t->cap + 1) * 4, ctx.compute);
  t->start = DevBuf(ctx.pool, (t->cap + 1) * 4, ctx.compute);
  t->rowidx = DevBuf(ctx.pool, std::max<uint64_t>(nb, 1) * 8, ctx.compute);
  DevBuf cursor(ctx.pool, (t->cap + 1) * 4, ctx.compute), maxc(ctx.pool, 4, ctx.compute),
      iota(ctx.pool, std::max<uint64_t>(nb, 1) * 8, ctx.compute);
  std::vector<uint64_t> seq(nb);
  std::iota(seq.begin(), seq.end(), 0ULL);
  if (nb) PSG_CUDA(cudaMemcpyAsync(iota.p, seq.data(), nb * 8, cudaMemcpyHostToDevice, ctx.compute));
  PSG_CUDA(cudaMemsetAsync(cursor.p, 0, (t->cap + 1) * 4, ctx.compute));
  PSG_CUDA(cudaMemsetAsync(maxc.p, 0, 4, ctx.compute));
  launch_local_init(t->keys.as<uint64_t>(), t->cnt.as<uint32_t>(), t->cap, ctx.compute);
  const uint64_t* bk = t->cols[t->key].as<uint64_t>();
  launch_local_count(t->keys.as<uint64_t>(), t->cnt.as<uint32_t>(), t->cap - 1, t->shift, bk, nb, maxc.as<unsigned>(),
                     ctx.compute);
  const size_t tb = exclusive_scan_u32(nullptr, nullptr, t->cap + 1, nullptr, 0, ctx.compute);
  DevBuf tmp(ctx.pool, tb, ctx.compute);
  exclusive_scan_u32(t->cnt.as<uint32_t>(), t->start.as<uint32_t>(), t->cap + 1, tmp.p, tb, ctx.compute);
  const uint64_t* src = iota.as<uint64_t>();
  uint64_t* dst = t->rowidx.as<uint64_t>();
  launch_local_fill(t->keys.as<uint64_t>(), t->start.as<uint32_t>(), cursor.as<uint32_t>(), t->cap - 1, t->shift, bk, &src,
                    &dst, 1, nb, ctx.compute);
  t->dev.keys = t->keys.as<uint64_t>();
  t->dev.cnt = t->cnt.as<uint32_t>();
  t->dev.start = t->start.as<uint32_t>();
  t->dev.mask = t->cap - 1;
  t->dev.shift = t->shift;
  t->dev.npayload = 1;  // CSR payload = build-row index
  t->dev.payload[0] = t->rowidx.as<uint64_t>();
  PSG_CUDA(cudaStreamSynchronize(ctx.compute));
  return t.release();
}

void op_hashtable_free(GpuHashTable* t) { delete t; }
const HostBatch& op_hashtable_host(const GpuHashTable& t) { return t.host; }

std::vector<uint64_t> op_hashtable_lookup(Ctx& ctx, const GpuHashTable& t, const std::vector<int64_t>& keys,
                                          std::vector<uint64_t>& offsets) {
  PSG_CUDA(cudaSetDevice(ctx.device));
  const uint64_t n = keys.size();
  DevBuf dk(ctx.pool, std::max<uint64_t>(n, 1) * 8, ctx.compute);
  if (n) PSG_CUDA(cudaMemcpyAsync(dk.p, keys.data(), n * 8, cudaMemcpyHostToDevice, ctx.compute));
  DevBuf offs, rows;
  const uint64_t total = t.rows ? expand_rows(ctx, t, dk.as<uint64_t>(), n, offs, rows) : 0;
  offsets.assign(n + 1, 0);
  if (t.rows) {
    std::vector<uint32_t> o32(n + 1);
    PSG_CUDA(cudaMemcpyAsync(o32.data(), offs.p, (n + 1) * 4, cudaMemcpyDeviceToHost, ctx.compute));
    PSG_CUDA(cudaStreamSynchronize(ctx.compute));
    for (uint64_t i = 0; i <= n; ++i) offsets[i] = o32[i];
  }
  std::vector<uint64_t> out = total ? download(ctx, rows, total) : std::vector<uint64_t>{};
  PSG_CUDA(cudaStreamSynchronize(ctx.compute));
  return out;
}

HostBatch op_hashtable_probe(Ctx& ctx, const GpuHashTable& t, const HostBatch& probe, const std::string& probe_key) {
  PSG_CUDA(cudaSetDevice(ctx.device));
  check_batch(probe);
  const size_t pk = probe.schema.require(probe_key);
  if (probe.schema.fields[pk].type != LType::Int64) throw InvalidInput("probe key must be int64: " + probe_key);
  // output schema: build payload ++ probe columns, "_p" on a name clash (ops.cpp:193-200)
  HostBatch out;
  out.schema = t.payload_schema;
  for (auto f : probe.schema.fields) {
    if (out.schema.index_of(f.name)) f.name += "_p";
    out.schema.fields.push_back(f);
  }
  const int np = static_cast<int>(t.payload_schema.size()), nq = static_cast<int>(probe.schema.size());
  out.cols.resize(np + nq);
  const uint64_t npr = probe.rows();
  if (t.rows == 0 || npr == 0) return out;
  Uploaded up = upload(ctx, probe);
  DevBuf offs, rows;
  const uint64_t total = expand_rows(ctx, t, up.cols[pk].as<uint64_t>(), npr, offs, rows);
  if (total == 0) return out;
  // probe side: each probe row repeated per match (expand_write with the probe columns)
  std::vector<DevBuf> oc;
  std::vector<uint64_t*> ocols;
  std::vector<const uint64_t*> pcols;
  for (int q = 0; q < nq; ++q) pcols.push_back(up.cols[q].as<uint64_t>());
  DevBuf scratch(ctx.pool, total * 8, ctx.compute);
  ocols.push_back(scratch.as<uint64_t>());  // build-row indices again (payload 0)
  for (int q = 0; q < nq; ++q) {
    oc.emplace_back(ctx.pool, total * 8, ctx.compute);
    ocols.push_back(oc.back().as<uint64_t>());
  }
  launch_expand_write(t.dev, up.cols[pk].as<uint64_t>(), npr, offs.as<uint32_t>(), pcols.data(), nq, ocols.data(),
                      ctx.compute);
  // build payload gathered by row index
  std::vector<DevBuf> bc;
  std::vector<const uint64_t*> bsrc;
  std::vector<uint64_t*> bdst;
  for (size_t c = 0; c < t.schema.size(); ++c) {
    if (c == t.key) continue;
    bc.emplace_back(ctx.pool, total * 8, ctx.compute);
    bsrc.push_back(t.cols[c].as<uint64_t>());
    bdst.push_back(bc.back().as<uint64_t>());
  }
  for (size_t c0 = 0; c0 < bsrc.size(); c0 += kMaxIn)
    launch_gather64(bsrc.data() + c0, static_cast<int>(std::min<size_t>(kMaxIn, bsrc.size() - c0)),
                    scratch.as<uint64_t>(), total, bdst.data() + c0, ctx.compute);
  for (int c = 0; c < np; ++c) out.cols[c] = download(ctx, bc[c], total);
  for (int q = 0; q < nq; ++q) out.cols[np + q] = download(ctx, oc[q], total);
  PSG_CUDA(cudaStreamSynchronize(ctx.compute));
  return out;
}

HostBatch op_hash_join(Ctx& ctx, const HostBatch& build, const std::string& build_key, const HostBatch& probe,
                       const std::string& probe_key) {
  std::unique_ptr<GpuHashTable> t(op_hashtable_build(ctx, {build}, build_key));
  return op_hashtable_probe(ctx, *t, probe, probe_key);
}

/// concat (ops.cpp:80-98): batches of one schema into one batch, assembled in HBM by the copy
/// engine (one D2D copy per input column) and returned.
HostBatch op_concat(Ctx& ctx, const std::vector<HostBatch>& batches) {
  PSG_CUDA(cudaSetDevice(ctx.device));
  if (batches.empty()) throw InvalidInput("concat needs at least one batch");
  const Schema& sc = batches[0].schema;
  uint64_t total = 0;
  for (const auto& b : batches) {
    check_batch(b);
    bool same = b.schema.size() == sc.size();
    for (size_t c = 0; same && c < sc.size(); ++c)
      same = b.schema.fields[c].name == sc.fields[c].name && b.schema.fields[c].type == sc.fields[c].type;
    if (!same) throw InvalidInput("concat: batches have different schemas");
    total += b.rows();
  }
  HostBatch out;
  out.schema = sc;
  out.cols.resize(sc.size());
  std::vector<DevBuf> dcols;
  for (size_t c = 0; c < sc.size(); ++c) dcols.emplace_back(ctx.pool, std::max<uint64_t>(total, 1) * 8, ctx.compute);
  uint64_t at = 0;
  for (const auto& b : batches) {
    const uint64_t n = b.rows();
    for (size_t c = 0; c < sc.size() && n; ++c)
      PSG_CUDA(cudaMemcpyAsync(dcols[c].as<uint8_t>() + at * 8, b.cols[c].data(), n * 8, cudaMemcpyHostToDevice,
                               ctx.compute));
    at += n;
  }
  for (size_t c = 0; c < sc.size(); ++c) out.cols[c] = download(ctx, dcols[c], total);
  PSG_CUDA(cudaStreamSynchronize(ctx.compute));
  return out;
}

}  // namespace psg
