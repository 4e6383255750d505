// Device memory pool, footer cache and the chunked storage->HBM ingest pipeline.
#include <emmintrin.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <chrono>
#include <cstdlib>
#include <fstream>
#include <map>
#include <cstring>

#include "engine.hpp"

namespace psg {

// ----------------------------------------------------------------------------- DevicePool
namespace {
constexpr uint64_t kPoolCacheMax = 120ull << 30;  // keep at most this much idle device memory
size_t round_block(size_t b) {
  // 2 MiB granularity above 64 MiB, 64 KiB below, so repeated queries hit identical sizes
  const size_t g = b >= (64u << 20) ? (2u << 20) : (64u << 10);
  return (b + g - 1) / g * g;
}
}  // namespace

void DevicePool::init(int device, uint64_t budget) {
  (void)device;
  budget_ = budget;
}

void* DevicePool::alloc(size_t bytes, cudaStream_t s) {
  const size_t rb = round_block(bytes ? bytes : 8);
  if (budget_ && used_ + rb > budget_) throw MemoryExceeded(rb, used_, budget_);
  void* p = nullptr;
  size_t got = rb;
  // best fit among this stream's idle blocks of size [rb, 2 rb]
  auto it = free_.lower_bound({s, rb});
  if (it != free_.end() && it->first.first == s && it->first.second <= 2 * rb && !it->second.empty()) {
    got = it->first.second;
    p = it->second.back();
    it->second.pop_back();
    cached_ -= got;
    if (it->second.empty()) free_.erase(it);
  } else {
    cudaError_t e = cudaMalloc(&p, rb);
    if (e != cudaSuccess) {
      cudaGetLastError();
      release_cache();  // give idle blocks back and retry once
      e = cudaMalloc(&p, rb);
      if (e != cudaSuccess) {
        cudaGetLastError();
        throw Error(PSG_ERR_MEMORY_EXCEEDED,
                    "device allocation of " + std::to_string(rb) + " bytes failed: " + cudaGetErrorString(e));
      }
    }
  }
  live_[p] = got;
  used_ += got;
  if (used_ > peak_) peak_ = used_;
  return p;
}

void DevicePool::free(void* p, cudaStream_t s) {
  auto it = live_.find(p);
  if (it == live_.end()) return;
  const size_t n = it->second;
  used_ -= n;
  live_.erase(it);
  if (cached_ + n > kPoolCacheMax) {
    cudaStreamSynchronize(s);
    cudaFree(p);
    return;
  }
  free_[{s, n}].push_back(p);
  cached_ += n;
}

void DevicePool::release_cache() {
  if (free_.empty()) return;
  cudaDeviceSynchronize();
  for (auto& [k, v] : free_)
    for (void* p : v) cudaFree(p);
  free_.clear();
  cached_ = 0;
}

// ----------------------------------------------------------------------------- PinnedBlock
namespace {
std::mutex g_pin_mu;
std::multimap<size_t, void*> g_pin_free;  // cached blocks by size
size_t g_pin_cached = 0;
constexpr size_t kPinCacheMax = 8ull << 30;
}  // namespace

std::shared_ptr<PinnedBlock> PinnedBlock::get(size_t bytes) {
  bytes = (bytes + (1u << 20) - 1) & ~size_t((1u << 20) - 1);
  auto b = std::shared_ptr<PinnedBlock>(new PinnedBlock());
  {
    std::lock_guard<std::mutex> lk(g_pin_mu);
    auto it = g_pin_free.lower_bound(bytes);
    if (it != g_pin_free.end() && it->first <= 2 * bytes) {
      b->n_ = it->first;
      b->p_ = it->second;
      g_pin_cached -= it->first;
      g_pin_free.erase(it);
      return b;
    }
  }
  PSG_CUDA(cudaHostAlloc(&b->p_, bytes, cudaHostAllocDefault));
  b->n_ = bytes;
  return b;
}

PinnedBlock::~PinnedBlock() {
  if (!p_) return;
  std::lock_guard<std::mutex> lk(g_pin_mu);
  if (g_pin_cached + n_ <= kPinCacheMax) {
    g_pin_free.emplace(n_, p_);
    g_pin_cached += n_;
  } else {
    cudaFreeHost(p_);
  }
}

// ----------------------------------------------------------------------------- FooterCache
std::shared_ptr<const TableMeta> FooterCache::get(const std::string& path) {
  struct stat st;
  if (::stat(path.c_str(), &st) != 0) throw IoFailure("cannot stat: " + path);
  const std::pair<int64_t, uint64_t> stamp{static_cast<int64_t>(st.st_mtim.tv_sec) * 1000000000LL + st.st_mtim.tv_nsec,
                                           static_cast<uint64_t>(st.st_size)};
  {
    std::lock_guard<std::mutex> lk(mu_);
    auto it = map_.find(path);
    if (it != map_.end() && it->second.first == stamp) return it->second.second;
  }
  auto meta = std::make_shared<const TableMeta>(read_footer(path));
  std::lock_guard<std::mutex> lk(mu_);
  map_[path] = {stamp, meta};
  return meta;
}

// ----------------------------------------------------------------------------- FileMapCache
namespace {
/// Copy into pinned staging memory with non-temporal stores: the destination lines are not read
/// for ownership and do not displace the page-cache source from the CPU caches (one host-memory
/// pass fewer per byte than memcpy's cached stores at column-chunk sizes, which stay below glibc's
/// non-temporal threshold). dst must be 16-byte aligned (batch buffers pack chunks at 16 bytes).
void copy_nt(uint8_t* dst, const uint8_t* src, size_t n) {
  if (n < 4096 || (reinterpret_cast<uintptr_t>(dst) & 15) != 0) {
    std::memcpy(dst, src, n);
    return;
  }
  auto* d = reinterpret_cast<__m128i*>(dst);
  const auto* sp = reinterpret_cast<const __m128i*>(src);
  const size_t k = n / 64;
  for (size_t i = 0; i < k; ++i) {
    const __m128i a = _mm_loadu_si128(sp + 4 * i), b = _mm_loadu_si128(sp + 4 * i + 1);
    const __m128i c = _mm_loadu_si128(sp + 4 * i + 2), e = _mm_loadu_si128(sp + 4 * i + 3);
    _mm_stream_si128(d + 4 * i, a);
    _mm_stream_si128(d + 4 * i + 1, b);
    _mm_stream_si128(d + 4 * i + 2, c);
    _mm_stream_si128(d + 4 * i + 3, e);
  }
  std::memcpy(dst + k * 64, src + k * 64, n - k * 64);
}
}  // namespace

FileMapping::~FileMapping() {
  if (base) ::munmap(const_cast<uint8_t*>(base), bytes);
}

bool FileMapCache::enabled() {
  static const bool on = [] {
    const char* e = std::getenv("PSG_MMAP");
    return !(e && e[0] == '0');
  }();
  return on;
}

std::shared_ptr<const FileMapping> FileMapCache::get(const std::string& path) {
  struct stat st;
  if (::stat(path.c_str(), &st) != 0 || st.st_size <= 0) return nullptr;
  const std::pair<int64_t, uint64_t> stamp{static_cast<int64_t>(st.st_mtim.tv_sec) * 1000000000LL + st.st_mtim.tv_nsec,
                                           static_cast<uint64_t>(st.st_size)};
  std::lock_guard<std::mutex> lk(mu_);
  auto it = map_.find(path);
  if (it != map_.end() && it->second.first == stamp) return it->second.second;
  const int fd = ::open(path.c_str(), O_RDONLY);
  if (fd < 0) return nullptr;
  void* p = ::mmap(nullptr, static_cast<size_t>(st.st_size), PROT_READ, MAP_SHARED, fd, 0);
  ::close(fd);
  if (p == MAP_FAILED) return nullptr;
  auto m = std::make_shared<FileMapping>();
  m->base = static_cast<const uint8_t*>(p);
  m->bytes = static_cast<size_t>(st.st_size);
  map_[path] = {stamp, m};
  return m;
}

// ----------------------------------------------------------------------------- Ctx
void Ctx::ensure_pinned(int nslots, uint64_t slot_bytes) {
  if (static_cast<int>(pinned.size()) >= nslots && pinned_slot_bytes >= slot_bytes) return;
  for (void* p : pinned) cudaFreeHost(p);
  pinned.clear();
  for (int i = 0; i < nslots; ++i) {
    void* p = nullptr;
    PSG_CUDA(cudaHostAlloc(&p, slot_bytes, cudaHostAllocDefault));
    pinned.push_back(p);
  }
  pinned_slot_bytes = slot_bytes;
}

void Ctx::init_symmetric_heap(size_t bytes) {
  if (nranks < 2 || !nccl || bytes == 0) return;
  cudaIpcMemHandle_t mine;
  std::vector<cudaIpcMemHandle_t> all(nranks);
  bool ok = cudaMalloc(&symm, bytes) == cudaSuccess;
  if (ok) ok = cudaIpcGetMemHandle(&mine, symm) == cudaSuccess;
  // zeroed barrier flags: ordered before the handle all-gather below, so before any peer's first
  // barrier store into them
  if (ok) ok = cudaMemsetAsync(symm + bytes - kSymmReserve, 0, kSymmReserve, compute) == cudaSuccess;
  barrier_epoch = 0;
  if (!ok) {
    cudaGetLastError();
    std::memset(&mine, 0, sizeof mine);
  }
  // all-gather the handles (and each rank's ok flag) over NCCL
  const size_t hb = sizeof(cudaIpcMemHandle_t) + 8;
  std::vector<uint8_t> blob(hb, 0);
  std::memcpy(blob.data(), &mine, sizeof mine);
  blob[sizeof mine] = ok ? 1 : 0;
  void *d_in = nullptr, *d_out = nullptr;
  PSG_CUDA(cudaMalloc(&d_in, hb));
  PSG_CUDA(cudaMalloc(&d_out, hb * nranks));
  PSG_CUDA(cudaMemcpy(d_in, blob.data(), hb, cudaMemcpyHostToDevice));
  if (ncclAllGather(d_in, d_out, hb, ncclUint8, nccl, compute) != ncclSuccess) throw Error(PSG_ERR_NCCL, "handle all-gather");
  std::vector<uint8_t> got(hb * nranks);
  PSG_CUDA(cudaMemcpyAsync(got.data(), d_out, got.size(), cudaMemcpyDeviceToHost, compute));
  PSG_CUDA(cudaStreamSynchronize(compute));
  cudaFree(d_in);
  cudaFree(d_out);
  bool all_ok = true;
  for (int p = 0; p < nranks; ++p) all_ok = all_ok && got[p * hb + sizeof(cudaIpcMemHandle_t)] == 1;
  symm_peer.assign(nranks, nullptr);
  for (int p = 0; p < nranks && all_ok; ++p) {
    if (p == rank) {
      symm_peer[p] = symm;
      continue;
    }
    cudaIpcMemHandle_t h;
    std::memcpy(&h, got.data() + p * hb, sizeof h);
    void* ptr = nullptr;
    if (cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      cudaGetLastError();
      all_ok = false;
      break;
    }
    symm_peer[p] = static_cast<uint8_t*>(ptr);
  }
  // every rank must agree: a single failure anywhere disables the fused path everywhere
  int flag = all_ok ? 1 : 0;
  int* d_flag = nullptr;
  PSG_CUDA(cudaMalloc(&d_flag, sizeof(int)));
  PSG_CUDA(cudaMemcpy(d_flag, &flag, sizeof(int), cudaMemcpyHostToDevice));
  if (ncclAllReduce(d_flag, d_flag, 1, ncclInt32, ncclMin, nccl, compute) != ncclSuccess)
    throw Error(PSG_ERR_NCCL, "p2p vote");
  PSG_CUDA(cudaMemcpyAsync(&flag, d_flag, sizeof(int), cudaMemcpyDeviceToHost, compute));
  PSG_CUDA(cudaStreamSynchronize(compute));
  cudaFree(d_flag);
  symm_bytes = flag == 1 ? bytes : 0;
  if (flag != 1) free_symmetric_heap_local();
}

void Ctx::free_symmetric_heap_local() {
  for (int p = 0; p < static_cast<int>(symm_peer.size()); ++p)
    if (p != rank && symm_peer[p]) cudaIpcCloseMemHandle(symm_peer[p]);
  symm_peer.clear();
  if (symm) cudaFree(symm);
  symm = nullptr;
  symm_bytes = symm_top = 0;
}

void Ctx::free_symmetric_heap() {
  if (!symm && symm_peer.empty()) return;
  PSG_CUDA(cudaDeviceSynchronize());
  for (int p = 0; p < static_cast<int>(symm_peer.size()); ++p)
    if (p != rank && symm_peer[p]) cudaIpcCloseMemHandle(symm_peer[p]);
  symm_peer.clear();
  // every peer has unmapped this rank's heap before it is freed
  if (nccl) {
    int* d = nullptr;
    PSG_CUDA(cudaMalloc(&d, sizeof(int)));
    if (ncclAllReduce(d, d, 1, ncclInt32, ncclMax, nccl, compute) != ncclSuccess) throw Error(PSG_ERR_NCCL, "heap barrier");
    PSG_CUDA(cudaStreamSynchronize(compute));
    cudaFree(d);
  }
  if (symm) cudaFree(symm);
  symm = nullptr;
  symm_bytes = symm_top = 0;
}

unsigned long long* Ctx::ensure_host_words() {
  if (!host_words) {
    void* p = nullptr;
    PSG_CUDA(cudaHostAlloc(&p, 4096, cudaHostAllocMapped));
    host_words = static_cast<unsigned long long*>(p);
  }
  return host_words;
}

Ctx::~Ctx() {
  cudaSetDevice(device);
  if (host_words) cudaFreeHost(host_words);
  for (int p = 0; p < static_cast<int>(symm_peer.size()); ++p)
    if (p != rank && symm_peer[p]) cudaIpcCloseMemHandle(symm_peer[p]);
  if (symm) cudaFree(symm);
  for (void* p : pinned) cudaFreeHost(p);
  if (nccl) ncclCommDestroy(nccl);
  if (ev_a) cudaEventDestroy(ev_a);
  if (ev_b) cudaEventDestroy(ev_b);
  if (compute) cudaStreamDestroy(compute);
  if (copy) cudaStreamDestroy(copy);
  if (comm) cudaStreamDestroy(comm);
}

// ----------------------------------------------------------------------------- Ingest
Ingest::Ingest(Ctx& ctx, const std::vector<std::string>& files, const std::vector<BatchPlan>& batches, int threads,
               uint64_t slot_bytes, int nslots)
    : ctx_(ctx), files_(files), batches_(batches), slot_bytes_(slot_bytes) {
  for (auto& f : files_) {
    const int fd = ::open(f.c_str(), O_RDONLY);
    if (fd < 0) {
      for (int x : fds_) ::close(x);
      throw IoFailure("cannot open: " + f);
    }
    ::posix_fadvise(fd, 0, 0, POSIX_FADV_SEQUENTIAL);
    fds_.push_back(fd);
    maps_.push_back(FileMapCache::enabled() ? ctx.maps.get(f) : nullptr);
  }
  ctx.ensure_pinned(nslots, slot_bytes);
  PSG_CUDA(cudaStreamCreateWithFlags(&cb_stream_, cudaStreamNonBlocking));
  slot_ev_.resize(nslots);
  for (auto& e : slot_ev_) PSG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  slots_.resize(nslots);
  for (int i = 0; i < nslots; ++i) {
    slots_[i].host = ctx.pinned[i];
    free_slots_.push_back(i);
  }
  slot_of_batch_.assign(batches.size(), -1);
  pending_.assign(batches.size(), 0);
  for (int t = 0; t < threads; ++t) threads_.emplace_back([this] { worker(); });
}

Ingest::~Ingest() {
  {
    std::lock_guard<std::mutex> lk(mu_);
    stop_ = true;
    cv_.notify_all();
  }
  for (auto& t : threads_) t.join();
  // Outstanding copies reference pinned slots; the caller synchronised the copy stream. The
  // release callbacks reference this object: drain their stream first.
  if (cb_stream_) {
    cudaStreamSynchronize(cb_stream_);
    cudaStreamDestroy(cb_stream_);
  }
  for (auto e : slot_ev_) cudaEventDestroy(e);
  for (int fd : fds_) ::close(fd);
}

void Ingest::worker() {
  // Readers share batches piece by piece (consecutive extents of >= kPiece bytes), in batch order:
  // the first batches are ready after 1/threads of their read time (a whole 128 MB batch per
  // thread delayed the first H2D copy by ~20 ms), and a batch's slot is taken when its first piece
  // is claimed.
  constexpr uint64_t kPiece = 16ull << 20;
  while (true) {
    size_t bi, e0, e1;
    int slot;
    {
      std::unique_lock<std::mutex> lk(mu_);
      auto open_left = [&] { return cur_batch_ >= 0 && cur_ext_ < batches_[cur_batch_].extents.size(); };
      cv_.wait(lk, [&] { return stop_ || open_left() || (next_job_ < batches_.size() && !free_slots_.empty()) ||
                                (!open_left() && next_job_ >= batches_.size()); });
      if (stop_) return;
      if (!open_left()) {
        if (next_job_ >= batches_.size()) return;
        bi = next_job_++;
        slot = free_slots_.front();
        free_slots_.pop_front();
        slots_[slot].batch = static_cast<int>(bi);
        slots_[slot].ready = false;
        slot_of_batch_[bi] = slot;
        pending_[bi] = 0;
        cur_batch_ = static_cast<long>(bi);
        cur_ext_ = 0;
        if (batches_[bi].extents.empty()) {  // nothing to read
          slots_[slot].ready = true;
          cv_.notify_all();
          continue;
        }
      }
      bi = static_cast<size_t>(cur_batch_);
      slot = slot_of_batch_[bi];
      const auto& ex = batches_[bi].extents;
      e0 = cur_ext_;
      uint64_t n = 0;
      while (cur_ext_ < ex.size() && n < kPiece) n += ex[cur_ext_++].len;
      e1 = cur_ext_;
      ++pending_[bi];
    }
    const BatchPlan& b = batches_[bi];
    auto* dst = static_cast<uint8_t*>(slots_[slot].host);
    std::string err;
    const auto t_read = std::chrono::steady_clock::now();
    const FileMapping* m = maps_[b.file].get();
    for (size_t x = e0; x < e1; ++x) {
      const Extent& e = b.extents[x];
      if (m != nullptr && e.file_off + e.len <= m->bytes) {  // straight out of the page cache
        copy_nt(dst + e.buf_off, m->base + e.file_off, e.len);
        continue;
      }
      uint64_t got = 0;
      while (got < e.len) {
        const ssize_t k = ::pread(fds_[b.file], dst + e.buf_off + got, e.len - got, static_cast<off_t>(e.file_off + got));
        if (k <= 0) {
          err = "short read of " + files_[b.file];
          break;
        }
        got += static_cast<uint64_t>(k);
      }
      if (!err.empty()) break;
    }
    _mm_sfence();  // the non-temporal stores are visible before the batch is marked ready
    if (ctx_.timeline) ctx_.timeline->host("read b" + std::to_string(bi), 0, t_read, std::chrono::steady_clock::now());
    std::lock_guard<std::mutex> lk(mu_);
    if (!err.empty() && error_.empty()) error_ = err;
    if (--pending_[bi] == 0 && !(cur_batch_ == static_cast<long>(bi) && cur_ext_ < b.extents.size())) {
      bytes_read_ += b.bytes;
      slots_[slot].ready = true;
      cv_.notify_all();
    }
  }
}

void CUDART_CB Ingest::on_copied(void* arg) {
  auto* d = static_cast<CopyDone*>(arg);
  std::lock_guard<std::mutex> lk(d->self->mu_);
  d->self->slots_[d->slot].batch = -1;
  d->self->free_slots_.push_back(d->slot);
  d->self->cv_.notify_all();
}

bool Ingest::ready(size_t i) {
  std::lock_guard<std::mutex> lk(mu_);
  return !error_.empty() || (slot_of_batch_[i] >= 0 && slots_[slot_of_batch_[i]].ready);
}

void Ingest::copy_to_device(size_t i, void* dst, const void* extra, size_t extra_bytes, cudaStream_t copy_stream) {
  int slot;
  {
    const auto t0 = std::chrono::steady_clock::now();
    std::unique_lock<std::mutex> lk(mu_);
    cv_.wait(lk, [&] { return !error_.empty() || (slot_of_batch_[i] >= 0 && slots_[slot_of_batch_[i]].ready); });
    wait_s_ += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (!error_.empty()) throw IoFailure(error_);
    slot = slot_of_batch_[i];
  }
  const BatchPlan& b = batches_[i];
  if (b.bytes + extra_bytes > slot_bytes_) throw InvalidInput("batch exceeds pinned slot size");
  auto* host = static_cast<uint8_t*>(slots_[slot].host);
  if (extra_bytes) std::memcpy(host + b.bytes, extra, extra_bytes);
  const int tl = ctx_.timeline ? ctx_.timeline->gpu_begin("h2d b" + std::to_string(i), 1, copy_stream) : -1;
  PSG_CUDA(cudaMemcpyAsync(dst, host, b.bytes + extra_bytes, cudaMemcpyHostToDevice, copy_stream));
  if (tl >= 0) ctx_.timeline->gpu_end(tl, copy_stream);
  done_args_.push_back(std::make_unique<CopyDone>(CopyDone{this, slot}));
  // The slot-release callback runs on a side stream that waits for the copy: a host function in
  // the copy stream itself holds back the NEXT copy until the host has run it (~0.4 ms between
  // every two 128 MB copies in the SF100 timeline: 14% of the end-to-end query).
  PSG_CUDA(cudaEventRecord(slot_ev_[slot], copy_stream));
  PSG_CUDA(cudaStreamWaitEvent(cb_stream_, slot_ev_[slot], 0));
  PSG_CUDA(cudaLaunchHostFunc(cb_stream_, &Ingest::on_copied, done_args_.back().get()));
}

// ----------------------------------------------------------------------------- Timeline
bool Timeline::enabled() {
  static const bool on = std::getenv("PSG_TIMELINE") != nullptr;
  return on;
}

Timeline::Timeline(cudaStream_t s) {
  PSG_CUDA(cudaEventCreate(&origin_));
  PSG_CUDA(cudaEventRecord(origin_, s));
  PSG_CUDA(cudaEventSynchronize(origin_));
  host_origin_ = std::chrono::steady_clock::now();
}

Timeline::~Timeline() {
  for (auto& g : gpu_) {
    cudaEventDestroy(g.a);
    cudaEventDestroy(g.b);
  }
  if (origin_) cudaEventDestroy(origin_);
}

int Timeline::gpu_begin(const std::string& name, int lane, cudaStream_t s) {
  Gpu g{name, lane, nullptr, nullptr};
  PSG_CUDA(cudaEventCreate(&g.a));
  PSG_CUDA(cudaEventCreate(&g.b));
  PSG_CUDA(cudaEventRecord(g.a, s));
  std::lock_guard<std::mutex> lk(mu_);
  gpu_.push_back(g);
  return static_cast<int>(gpu_.size() - 1);
}

void Timeline::gpu_end(int id, cudaStream_t s) {
  cudaEvent_t b;
  {
    std::lock_guard<std::mutex> lk(mu_);
    b = gpu_[id].b;
  }
  PSG_CUDA(cudaEventRecord(b, s));
}

void Timeline::host(const std::string& name, int lane, std::chrono::steady_clock::time_point a,
                    std::chrono::steady_clock::time_point b) {
  std::lock_guard<std::mutex> lk(mu_);
  host_.push_back({name, lane, std::chrono::duration<double, std::micro>(a - host_origin_).count(),
                   std::chrono::duration<double, std::micro>(b - host_origin_).count()});
}

void Timeline::dump(const std::string& path, int rank) {
  PSG_CUDA(cudaDeviceSynchronize());
  static const char* lanes[] = {"host reads", "H2D copy", "inflate", "compute", "exchange"};
  std::ofstream out(path + ".rank" + std::to_string(rank) + ".json");
  out << "{\"traceEvents\": [\n";
  bool first = true;
  auto emit = [&](const std::string& name, int lane, double a, double b) {
    if (b < a) return;
    out << (first ? "" : ",\n") << "{\"name\": \"" << name << "\", \"ph\": \"X\", \"pid\": " << rank
        << ", \"tid\": " << lane << ", \"ts\": " << a << ", \"dur\": " << (b - a) << "}";
    first = false;
  };
  for (int l = 0; l < 5; ++l) {
    out << (first ? "" : ",\n") << "{\"name\": \"thread_name\", \"ph\": \"M\", \"pid\": " << rank
        << ", \"tid\": " << l << ", \"args\": {\"name\": \"" << lanes[l] << "\"}}";
    first = false;
  }
  for (auto& g : gpu_) {
    float a = 0, b = 0;
    if (cudaEventElapsedTime(&a, origin_, g.a) != cudaSuccess || cudaEventElapsedTime(&b, origin_, g.b) != cudaSuccess) {
      cudaGetLastError();
      continue;
    }
    emit(g.name, g.lane, a * 1000.0, b * 1000.0);
  }
  for (auto& h : host_) emit(h.name, h.lane, h.a_us, h.b_us);
  out << "\n]}\n";
}

}  // namespace psg
