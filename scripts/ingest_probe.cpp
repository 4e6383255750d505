// Measurement tool (not product code): host->HBM ingest capabilities of the box.
//   ingest_probe <file>...            (files should be in the page cache: warm)
// Prints GB/s for: pread into pinned buffers with T threads (no GPU), pinned H2D copies,
// and mmap + cudaHostRegister + H2D (DMA straight from page-cache pages).
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <atomic>
#include <mutex>
#include <chrono>
#include <cstdio>
#include <string>
#include <thread>
#include <vector>

using Clock = std::chrono::steady_clock;
static double since(Clock::time_point t) { return std::chrono::duration<double>(Clock::now() - t).count(); }

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
  // ---- 1. pread into pinned memory, T threads, chunk jobs round robin
  for (int T : {4, 8, 16, 32}) {
    std::vector<void*> bufs(T);
    for (auto& b : bufs) cudaHostAlloc(&b, chunk, 0);
    std::atomic<size_t> next{0};
    std::vector<std::pair<int, size_t>> jobs;
    for (size_t f = 0; f < files.size(); ++f)
      for (size_t off = 0; off < sizes[f]; off += chunk) jobs.push_back({(int)f, off});
    std::vector<int> fds;
    for (auto& f : files) fds.push_back(open(f.c_str(), O_RDONLY));
    auto t0 = Clock::now();
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t)
      th.emplace_back([&, t] {
        size_t j;
        while ((j = next++) < jobs.size()) {
          auto [f, off] = jobs[j];
          size_t len = std::min(chunk, sizes[f] - off), got = 0;
          while (got < len) {
            ssize_t k = pread(fds[f], (char*)bufs[t] + got, len - got, off + got);
            if (k <= 0) break;
            got += k;
          }
        }
      });
    for (auto& x : th) x.join();
    double s = since(t0);
    std::fflush(stdout), std::printf("pread->pinned T=%2d: %.2f GB in %.3f s = %.1f GB/s\n", T, total / 1e9, s, total / 1e9 / s);
    for (int fd : fds) close(fd);
    for (auto& b : bufs) cudaFreeHost(b);
  }
  // ---- 2. pinned H2D
  {
    void *h, *d;
    cudaHostAlloc(&h, chunk, 0);
    cudaMalloc(&d, 1ull << 30);
    cudaStream_t s[2];
    cudaStreamCreate(&s[0]);
    cudaStreamCreate(&s[1]);
    for (int ns : {1, 2}) {
      cudaDeviceSynchronize();
      auto t0 = Clock::now();
      const int n = 200;
      for (int i = 0; i < n; ++i)
        cudaMemcpyAsync((char*)d + (i % 16) * chunk, h, chunk, cudaMemcpyHostToDevice, s[i % ns]);
      cudaDeviceSynchronize();
      double sec = since(t0);
      std::fflush(stdout), std::printf("pinned H2D 64MB x %d, %d stream(s): %.1f GB/s\n", n, ns, n * chunk / 1e9 / sec);
    }
    cudaFreeHost(h);
    cudaFree(d);
  }
  // ---- 3. page-cache pages registered with the GPU (zero-copy DMA), several variants
  {
    int dev = 0, ro = 0;
    cudaDeviceGetAttribute(&ro, cudaDevAttrHostRegisterReadOnlySupported, dev);
    std::fflush(stdout), std::printf("cudaDevAttrHostRegisterReadOnlySupported = %d\n", ro);
    void* d;
    cudaMalloc(&d, chunk);
    struct Var { const char* name; int oflag, prot, mflag; unsigned reg; };
    Var vars[] = {{"shared ro + ReadOnly", O_RDONLY, PROT_READ, MAP_SHARED, cudaHostRegisterReadOnly},
                  {"shared rw + Default", O_RDWR, PROT_READ | PROT_WRITE, MAP_SHARED, cudaHostRegisterDefault},
                  {"shared ro + Default", O_RDONLY, PROT_READ, MAP_SHARED, cudaHostRegisterDefault}};
    for (auto& v : vars) {
      size_t done = 0;
      double reg_s = 0, copy_s = 0;
      bool ok = true;
      for (size_t f = 0; f < files.size() && done < (6ull << 30); ++f) {
        int fd = open(files[f].c_str(), v.oflag);
        void* p = mmap(nullptr, sizes[f], v.prot, v.mflag | MAP_POPULATE, fd, 0);
        if (p == MAP_FAILED) { std::fflush(stdout), std::printf("%s: mmap failed\n", v.name); ok = false; close(fd); break; }
        auto t0 = Clock::now();
        cudaError_t e = cudaHostRegister(p, sizes[f], v.reg);
        reg_s += since(t0);
        if (e != cudaSuccess) {
          std::fflush(stdout), std::printf("%s: cudaHostRegister failed: %s\n", v.name, cudaGetErrorString(e));
          cudaGetLastError();
          munmap(p, sizes[f]);
          close(fd);
          ok = false;
          break;
        }
        t0 = Clock::now();
        for (size_t off = 0; off < sizes[f]; off += chunk)
          cudaMemcpyAsync(d, (char*)p + off, std::min(chunk, sizes[f] - off), cudaMemcpyHostToDevice, 0);
        cudaDeviceSynchronize();
        copy_s += since(t0);
        done += sizes[f];
        cudaHostUnregister(p);
        munmap(p, sizes[f]);
        close(fd);
      }
      if (ok && done)
        std::fflush(stdout), std::printf("%s: %.2f GB register %.3f s (%.1f GB/s), H2D %.3f s (%.1f GB/s)\n", v.name, done / 1e9, reg_s,
                    done / 1e9 / reg_s, copy_s, done / 1e9 / copy_s);
    }
    cudaFree(d);
  }
  // ---- 4. pread->pinned overlapped with pinned H2D (the engine's pattern): T readers + 1 copier
  for (int T : {8, 16, 24}) {
    const int nslots = 2 * T + 2;
    std::vector<void*> bufs(nslots);
    for (auto& b : bufs) cudaHostAlloc(&b, chunk, 0);
    void* d;
    cudaMalloc(&d, chunk);
    std::vector<std::pair<int, size_t>> jobs;
    for (size_t f = 0; f < files.size(); ++f)
      for (size_t off = 0; off < sizes[f]; off += chunk) jobs.push_back({(int)f, off});
    std::vector<int> fds;
    for (auto& f : files) fds.push_back(open(f.c_str(), O_RDONLY));
    std::vector<std::atomic<int>> state(nslots);  // 0 free, 1 reading, 2 ready
    for (auto& s2 : state) s2 = 0;
    std::vector<int> slot_of(jobs.size(), -1);
    std::atomic<size_t> next{0};
    std::atomic<int> ready_count{0};
    auto t0 = Clock::now();
    std::vector<std::thread> th;
    std::vector<std::atomic<int>> done(jobs.size());
    for (auto& x : done) x = 0;
    std::mutex claim_mu;
    for (int t = 0; t < T; ++t)
      th.emplace_back([&] {
        while (true) {
          // claim the next job together with a free slot, in job order (no in-order deadlock)
          size_t j;
          int s2 = -1;
          while (true) {
            std::lock_guard<std::mutex> lk(claim_mu);
            if (next >= jobs.size()) return;
            for (int k = 0; k < nslots && s2 < 0; ++k) {
              int z = 0;
              if (state[k].compare_exchange_strong(z, 1)) s2 = k;
            }
            if (s2 >= 0) {
              j = next++;
              break;
            }
          }
          auto [f, off] = jobs[j];
          size_t len = std::min(chunk, sizes[f] - off), got = 0;
          while (got < len) {
            ssize_t k = pread(fds[f], (char*)bufs[s2] + got, len - got, off + got);
            if (k <= 0) break;
            got += k;
          }
          slot_of[j] = s2;
          done[j] = 1;
        }
      });
    cudaStream_t st;
    cudaStreamCreate(&st);
    std::vector<cudaEvent_t> evs(nslots);
    for (auto& e : evs) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    std::vector<int> inflight;  // slots with pending copies
    for (size_t j = 0; j < jobs.size(); ++j) {
      while (!done[j]) {
        // retire finished copies
        for (size_t q = 0; q < inflight.size();) {
          if (cudaEventQuery(evs[inflight[q]]) == cudaSuccess) { state[inflight[q]] = 0; inflight.erase(inflight.begin() + q); }
          else ++q;
        }
      }
      int s2 = slot_of[j];
      auto [f, off] = jobs[j];
      cudaMemcpyAsync(d, bufs[s2], std::min(chunk, sizes[f] - off), cudaMemcpyHostToDevice, st);
      cudaEventRecord(evs[s2], st);
      inflight.push_back(s2);
    }
    cudaStreamSynchronize(st);
    for (auto& x : th) x.join();
    double s = since(t0);
    std::fflush(stdout), std::printf("pipelined pread+H2D T=%2d: %.1f GB/s\n", T, total / 1e9 / s);
    for (int fd : fds) close(fd);
    for (auto& b : bufs) cudaFreeHost(b);
    cudaFree(d);
  }
  return 0;
}
