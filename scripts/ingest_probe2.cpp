// Measurement tool (not product code): ways around the page cache -> pinned copy of the ingest.
//   ingest_probe2 <file>...   (warm page cache)
// 1. cudaHostRegister of PRIVATE read-only file mappings and of a /dev/shm (shmem) copy.
// 2. mmap'd files (mapping kept, MAP_POPULATE) copied into pinned slots by T threads with
//    non-temporal 16-byte stores (no read-for-ownership of the destination), pipelined with the
//    H2D copies of one copy stream - vs the same pipeline with pread (the engine's pattern).
#include <cuda_runtime.h>
#include <emmintrin.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

using Clock = std::chrono::steady_clock;
static double since(Clock::time_point t) { return std::chrono::duration<double>(Clock::now() - t).count(); }

static void nt_copy(void* dst, const void* src, size_t n) {
  auto* d = static_cast<__m128i*>(dst);
  auto* s = static_cast<const __m128i*>(src);
  size_t k = n / 64;
  for (size_t i = 0; i < k; ++i) {
    __m128i a = _mm_loadu_si128(s + 4 * i), b = _mm_loadu_si128(s + 4 * i + 1);
    __m128i c = _mm_loadu_si128(s + 4 * i + 2), e = _mm_loadu_si128(s + 4 * i + 3);
    _mm_stream_si128(d + 4 * i, a);
    _mm_stream_si128(d + 4 * i + 1, b);
    _mm_stream_si128(d + 4 * i + 2, c);
    _mm_stream_si128(d + 4 * i + 3, e);
  }
  std::memcpy(reinterpret_cast<char*>(dst) + k * 64, reinterpret_cast<const char*>(src) + k * 64, n - k * 64);
  _mm_sfence();
}

int main(int argc, char** argv) {
  std::vector<std::string> files(argv + 1, argv + argc);
  std::vector<size_t> sizes;
  size_t total = 0;
  for (auto& f : files) {
    struct stat st;
    stat(f.c_str(), &st);
    sizes.push_back(st.st_size);
    total += st.st_size;
  }
  const size_t chunk = 64ull << 20;
  // ---- 1. registration variants
  {
    struct Var { const char* name; int mflag; unsigned reg; };
    Var vars[] = {{"private ro + ReadOnly", MAP_PRIVATE, cudaHostRegisterReadOnly},
                  {"private ro + Default", MAP_PRIVATE, cudaHostRegisterDefault}};
    for (auto& v : vars) {
      int fd = open(files[0].c_str(), O_RDONLY);
      void* p = mmap(nullptr, sizes[0], PROT_READ, v.mflag | MAP_POPULATE, fd, 0);
      auto t0 = Clock::now();
      cudaError_t e = cudaHostRegister(p, sizes[0], v.reg);
      std::printf("%s: %s (%.3f s for %.2f GB)\n", v.name, cudaGetErrorString(e), since(t0), sizes[0] / 1e9);
      cudaGetLastError();
      if (e == cudaSuccess) cudaHostUnregister(p);
      munmap(p, sizes[0]);
      close(fd);
    }
    // shmem-backed file
    const char* shm = "/dev/shm/psg_probe.bin";
    int in = open(files[0].c_str(), O_RDONLY), out = open(shm, O_RDWR | O_CREAT | O_TRUNC, 0600);
    size_t n = std::min<size_t>(sizes[0], 2ull << 30);
    std::vector<char> buf(chunk);
    for (size_t off = 0; off < n; off += chunk) {
      ssize_t k = pread(in, buf.data(), std::min(chunk, n - off), off);
      if (k <= 0 || write(out, buf.data(), k) != k) break;
    }
    close(in);
    void* p = mmap(nullptr, n, PROT_READ, MAP_SHARED | MAP_POPULATE, out, 0);
    for (unsigned reg : {(unsigned)cudaHostRegisterReadOnly, (unsigned)cudaHostRegisterDefault}) {
      auto t0 = Clock::now();
      cudaError_t e = cudaHostRegister(p, n, reg);
      std::printf("/dev/shm shared ro + %s: %s (%.3f s for %.2f GB)\n", reg ? "ReadOnly" : "Default", cudaGetErrorString(e),
                  since(t0), n / 1e9);
      cudaGetLastError();
      if (e == cudaSuccess) {
        void* d;
        cudaMalloc(&d, chunk);
        t0 = Clock::now();
        for (int r = 0; r < 3; ++r)
          for (size_t off = 0; off < n; off += chunk) cudaMemcpyAsync(d, (char*)p + off, std::min(chunk, n - off), cudaMemcpyHostToDevice, 0);
        cudaDeviceSynchronize();
        std::printf("  H2D from registered shmem: %.1f GB/s\n", 3 * n / 1e9 / since(t0));
        cudaFree(d);
        cudaHostUnregister(p);
      }
    }
    munmap(p, n);
    close(out);
    unlink(shm);
  }
  // ---- 2. pipelined copy + H2D: pread vs NT copy from kept mappings
  std::vector<const char*> maps(files.size());
  {
    auto t0 = Clock::now();
    for (size_t f = 0; f < files.size(); ++f) {
      int fd = open(files[f].c_str(), O_RDONLY);
      maps[f] = static_cast<const char*>(mmap(nullptr, sizes[f], PROT_READ, MAP_SHARED | MAP_POPULATE, fd, 0));
      madvise(const_cast<char*>(maps[f]), sizes[f], MADV_HUGEPAGE);
      close(fd);
    }
    std::printf("mmap+populate of %.2f GB: %.3f s\n", total / 1e9, since(t0));
  }
  std::vector<std::pair<int, size_t>> jobs;
  for (size_t f = 0; f < files.size(); ++f)
    for (size_t off = 0; off < sizes[f]; off += chunk) jobs.push_back({(int)f, off});
  std::vector<int> fds;
  for (auto& f : files) fds.push_back(open(f.c_str(), O_RDONLY));
  for (int mode = 0; mode < 3; ++mode)  // 0 pread, 1 NT copy from mapping, 2 memcpy from mapping
    for (int T : {8, 12, 16}) {
      // copy alone (no DMA)
      const int nslots = 2 * T + 2;
      std::vector<void*> bufs(nslots);
      for (auto& b : bufs) cudaHostAlloc(&b, chunk, 0);
      auto fill = [&](size_t j, void* dst) {
        auto [f, off] = jobs[j];
        size_t len = std::min(chunk, sizes[f] - off);
        if (mode == 0) {
          size_t got = 0;
          while (got < len) {
            ssize_t k = pread(fds[f], (char*)dst + got, len - got, off + got);
            if (k <= 0) break;
            got += k;
          }
        } else if (mode == 1) {
          nt_copy(dst, maps[f] + off, len);
        } else {
          std::memcpy(dst, maps[f] + off, len);
        }
      };
      {
        std::atomic<size_t> next{0};
        auto t0 = Clock::now();
        std::vector<std::thread> th;
        for (int t = 0; t < T; ++t)
          th.emplace_back([&, t] {
            size_t j;
            while ((j = next++) < jobs.size()) fill(j, bufs[t]);
          });
        for (auto& x : th) x.join();
        std::printf("%s T=%2d copy only: %.1f GB/s\n", mode == 0 ? "pread " : mode == 1 ? "ntcopy" : "memcpy", T,
                    total / 1e9 / since(t0));
      }
      void* d;
      cudaMalloc(&d, chunk);
      cudaStream_t st;
      cudaStreamCreate(&st);
      std::vector<cudaEvent_t> evs(nslots);
      for (auto& e : evs) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
      std::vector<std::atomic<int>> state(nslots);  // 0 free, 1 filling
      for (auto& s : state) s = 0;
      std::vector<std::atomic<int>> slot_of(jobs.size());
      for (auto& s : slot_of) s = -1;
      std::atomic<size_t> next{0};
      auto t0 = Clock::now();
      std::vector<std::thread> th;
      for (int t = 0; t < T; ++t)
        th.emplace_back([&] {
          while (true) {
            // slot first, then the job: the oldest unfilled job always holds a slot
            int s = -1;
            while (s < 0) {
              if (next >= jobs.size()) return;
              for (int k = 0; k < nslots && s < 0; ++k) {
                int z = 0;
                if (state[k].compare_exchange_strong(z, 1)) s = k;
              }
            }
            size_t j = next++;
            if (j >= jobs.size()) { state[s] = 0; return; }
            fill(j, bufs[s]);
            slot_of[j] = s;
          }
        });
      std::vector<int> inflight;
      for (size_t j = 0; j < jobs.size(); ++j) {
        while (slot_of[j] < 0)
          for (size_t q = 0; q < inflight.size();) {
            if (cudaEventQuery(evs[inflight[q]]) == cudaSuccess) {
              state[inflight[q]] = 0;
              inflight.erase(inflight.begin() + q);
            } else {
              ++q;
            }
          }
        int s = slot_of[j];
        auto [f, off] = jobs[j];
        cudaMemcpyAsync(d, bufs[s], std::min(chunk, sizes[f] - off), cudaMemcpyHostToDevice, st);
        cudaEventRecord(evs[s], st);
        inflight.push_back(s);
      }
      cudaStreamSynchronize(st);
      for (int s : inflight) state[s] = 0;
      for (auto& x : th) x.join();
      std::printf("%s T=%2d pipelined with H2D: %.1f GB/s\n", mode == 0 ? "pread " : mode == 1 ? "ntcopy" : "memcpy", T,
                  total / 1e9 / since(t0));
      for (auto& e : evs) cudaEventDestroy(e);
      cudaStreamDestroy(st);
      cudaFree(d);
      for (auto& b : bufs) cudaFreeHost(b);
    }
  return 0;
}
