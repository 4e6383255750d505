// GPU inflate for the PSTO block codec (zlib streams, deflate level 1 at write time).
//
// The reference decodes every compressed column chunk on the host with zlib's uncompress
// (codec_decompress, psto.cpp:133-143, called per chunk from decode_group, scan.cpp:139-160) and
// raises IoFailure("inflate failed") on any error or size mismatch. Here the compressed chunks
// travel host->HBM as they are (3-8x fewer PCIe bytes than decoded columns) and are expanded in
// HBM by this kernel, straight into the chunk layout the fused scan kernel reads.
//
// Design (B200): a deflate stream is inherently serial, so parallelism comes from chunks - one
// thread decodes one chunk (a 256 KB column chunk is ~30-100 KB of stream) and an SM keeps 256
// decoders in flight. Per-thread state:
//   * bit reader: 64-bit buffer refilled with aligned 32-bit loads (chunks are 16-byte aligned);
//   * Huffman tables in shared memory, laid out [entry][thread] so a warp's lookups are
//     bank-conflict free whatever entries the lanes hit; decoding is branch-free canonical:
//     the 15 left-justified per-length limits live in registers, code length = 1 + #limits <=
//     the bit-reversed peek, symbol = sym[base[len] + (peek >> (15 - len))];
//   * output is assembled in a 64-bit register and written as aligned 8-byte stores; matches
//     with distance >= 8 copy 8 bytes per step (two aligned loads + funnel shift, the newest
//     bytes taken from the register), shorter distances byte by byte;
//   * Adler-32 of the output is folded in per 8-byte word with dp4a (zlib verifies it too).
// Every failure zlib reports (bad header, bad block type, over-subscribed/incomplete codes,
// invalid symbols, distance too far back, output overrun or short output, input overrun, Adler
// mismatch) sets the job's error word; the host turns it into IoFailure("inflate failed").
#include <algorithm>
#include <cstdint>

#include "kernels.cuh"

namespace psg {
namespace {

constexpr int kThreads = 64;   // decoders per CTA; 48 KB of tables per CTA -> 4 CTAs per SM
constexpr int kLitSyms = 288;  // literal/length alphabet (fixed code uses all 288)
constexpr int kDistSyms = 32;  // distance alphabet (fixed code uses 32 five-bit codes)

__constant__ uint16_t c_lbase[29] = {3,  4,  5,  6,  7,  8,  9,  10, 11,  13,  15,  17,  19,  23, 27,
                                     31, 35, 43, 51, 59, 67, 83, 99, 115, 131, 163, 195, 227, 258};
__constant__ uint8_t c_lext[29] = {0, 0, 0, 0, 0, 0, 0, 0, 1, 1, 1, 1, 2, 2, 2, 2, 3, 3, 3, 3, 4, 4, 4, 4, 5, 5, 5, 5, 0};
__constant__ uint16_t c_dbase[30] = {1,   2,   3,   4,   5,   7,    9,    13,   17,   25,   33,   49,   65,    97,    129,
                                     193, 257, 385, 513, 769, 1025, 1537, 2049, 3073, 4097, 6145, 8193, 12289, 16385, 24577};
__constant__ uint8_t c_dext[30] = {0, 0, 0, 0, 1, 1, 2, 2, 3, 3, 4, 4, 5, 5, 6, 6, 7, 7, 8, 8, 9, 9, 10, 10, 11, 11, 12, 12, 13, 13};
__constant__ uint8_t c_clorder[19] = {16, 17, 18, 0, 8, 7, 9, 6, 10, 5, 11, 4, 12, 3, 13, 2, 14, 1, 15};

struct Smem {
  uint16_t lsym[kLitSyms][kThreads];
  uint16_t dsym[kDistSyms][kThreads];
  int32_t lbase[16][kThreads];
  int32_t dbase[16][kThreads];
};
static_assert(sizeof(Smem) <= 48 * 1024, "inflate tables exceed static shared memory");

/// Canonical Huffman table: limits in registers, base/sym in shared memory (column `t`).
/// Returns false for codes zlib rejects (inflate_table: over-subscribed, or incomplete unless it
/// is a single one-bit code of a literal/length or distance table).
__device__ __forceinline__ bool build_table(const uint8_t* lens, int n, bool code_lengths, uint16_t (*sym)[kThreads],
                                            int32_t (*base)[kThreads], uint32_t (&lim)[16], int t) {
  uint16_t cnt[16];
#pragma unroll
  for (int l = 0; l < 16; ++l) cnt[l] = 0;
  for (int i = 0; i < n; ++i) cnt[lens[i]]++;
  cnt[0] = 0;
  int maxlen = 0;
#pragma unroll
  for (int l = 1; l < 16; ++l)
    if (cnt[l]) maxlen = l;
  int left = 1;
#pragma unroll
  for (int l = 1; l < 16; ++l) {
    left <<= 1;
    left -= cnt[l];
    if (left < 0) return false;  // over-subscribed
  }
  if (maxlen > 0 && left > 0 && (code_lengths || maxlen != 1)) return false;  // incomplete
  uint16_t offs[16];
  uint32_t code = 0;
  int off = 0;
#pragma unroll
  for (int l = 1; l < 16; ++l) {
    offs[l] = static_cast<uint16_t>(off);
    base[l][t] = off - static_cast<int32_t>(code);
    lim[l] = (code + cnt[l]) << (15 - l);
    code = (code + cnt[l]) << 1;
    off += cnt[l];
  }
  for (int i = 0; i < n; ++i)
    if (lens[i]) sym[offs[lens[i]]++][t] = static_cast<uint16_t>(i);
  return true;
}

__device__ __forceinline__ uint64_t shl(uint64_t x, int s) { return s < 64 ? x << s : 0ull; }
__device__ __forceinline__ uint64_t low_bytes(uint64_t x, int k) { return k >= 8 ? x : x & ((1ull << (8 * k)) - 1ull); }

enum Mode : int { kIdle = 0, kSym = 1, kCopy = 2, kStart = 3, kHeader = 4, kStored = 5, kTrailer = 6 };

/// One decoder lane: bit reader, output assembler and the block state machine. Every call of
/// step() does a bounded amount of work - decode one symbol, or move <= 8 bytes of a match or
/// stored block - so the 32 lanes of a warp stay on the same instruction stream.
struct Lane {
  // ---- job
  const InflateJob* jobs;
  uint32_t njobs, j, stride;
  uint64_t usize;
  uint32_t csize;
  // ---- bit reader (LSB first); `nextw` is loaded one refill ahead to hide the load latency
  const uint32_t* p;
  const uint32_t* end;
  uint64_t b;
  int n;
  uint32_t nextw, loaded;
  // ---- output: bytes [0, oi) stored, `an` (< 8) pending in acc; w1/w2 = words at oi-8 / oi-16
  uint64_t* dst;
  uint64_t oi, acc, w1, w2;
  int an;
  uint32_t s1, s2;
  // ---- block state
  int mode;
  bool last;
  uint32_t rem, dist;
  uint32_t llim[16], dlim[16];

  __device__ __forceinline__ void refill() {
    if (n <= 32) {
      b |= static_cast<uint64_t>(nextw) << n;
      n += 32;
      ++loaded;
      nextw = p < end ? __ldg(p) : 0u;
      ++p;
    }
  }
  __device__ __forceinline__ uint32_t get(int k) {  // k <= 32 and n >= k
    const uint32_t v = static_cast<uint32_t>(b) & static_cast<uint32_t>((1ull << k) - 1ull);
    b >>= k;
    n -= k;
    return v;
  }
  __device__ __forceinline__ uint64_t consumed_bits() const { return static_cast<uint64_t>(loaded) * 32ull - n; }
  __device__ __forceinline__ uint64_t pos() const { return oi + an; }

  /// Decodes one symbol (>= 15 bits buffered); -1 for a code outside the table.
  __device__ __forceinline__ int decode(const uint32_t (&lim)[16], const uint16_t (*sym)[kThreads],
                                        const int32_t (*base)[kThreads], int t) {
    const uint32_t c15 = __brev(static_cast<uint32_t>(b)) >> 17;
    int len = 1;
#pragma unroll
    for (int l = 1; l < 16; ++l) len += (c15 >= lim[l]) ? 1 : 0;
    if (len > 15) return -1;
    const int idx = base[len][t] + static_cast<int>(c15 >> (15 - len));
    b >>= len;
    n -= len;
    return sym[idx][t];
  }

  __device__ __forceinline__ void flush_word(uint64_t w) {
    dst[oi >> 3] = w;
    const uint32_t lo = static_cast<uint32_t>(w), hi = static_cast<uint32_t>(w >> 32);
    s2 += 8u * s1 + __dp4a(lo, 0x05060708u, 0u) + __dp4a(hi, 0x01020304u, 0u);
    s1 += __dp4a(lo, 0x01010101u, 0u) + __dp4a(hi, 0x01010101u, 0u);
    if ((oi & 2047) == 2040) {  // every 256 words: keep s2 below 2^32
      s1 %= 65521u;
      s2 %= 65521u;
    }
    w2 = w1;
    w1 = w;
    oi += 8;
  }
  /// Appends the low k (1..8) bytes of v.
  __device__ __forceinline__ void put(uint64_t v, int k) {
    v = low_bytes(v, k);
    acc |= shl(v, 8 * an);
    const int t = an + k;
    if (t >= 8) {
      flush_word(acc);
      acc = an ? (v >> (64 - 8 * an)) : 0ull;
      an = t - 8;
    } else {
      an = t;
    }
  }
  /// 8 bytes at position s, s + 8 <= pos() (so s < oi): from the register window when recent.
  __device__ __forceinline__ uint64_t read8(uint64_t s) const {
    const int sh = static_cast<int>(s & 7) * 8;
    if (static_cast<int64_t>(s) >= static_cast<int64_t>(oi) - 16) {
      const bool q0 = s < oi - 8;  // starts in the w2 word
      const uint64_t lo = q0 ? w2 : w1, hi = q0 ? w1 : acc;
      return sh ? (lo >> sh) | (hi << (64 - sh)) : lo;
    }
    const uint64_t* m = dst + (s >> 3);
    const uint64_t a = m[0];
    return sh ? (a >> sh) | (m[1] << (64 - sh)) : a;
  }
  /// The 8 bytes ending at pos() (positions before 0 are never referenced).
  __device__ __forceinline__ uint64_t last8() const { return an ? (w1 >> (8 * an)) | (acc << (64 - 8 * an)) : w1; }

  __device__ __forceinline__ void fail(unsigned int* err) {
    atomicOr(err, 1u);
    j += stride;
    mode = kStart;
  }

  __device__ void start(unsigned int* err) {
    if (j >= njobs) {
      mode = kIdle;
      return;
    }
    const InflateJob job = jobs[j];
    usize = job.usize;
    csize = job.csize;
    p = reinterpret_cast<const uint32_t*>(job.src);
    end = p + (job.csize + 3) / 4;
    nextw = p < end ? __ldg(p) : 0u;
    ++p;
    loaded = 0;
    b = 0;
    n = 0;
    dst = reinterpret_cast<uint64_t*>(job.dst);
    oi = acc = w1 = w2 = 0;
    an = 0;
    s1 = 1;
    s2 = 0;
    last = false;
    refill();
    // zlib header (RFC 1950): deflate, window <= 32K, no preset dictionary, FCHECK
    const uint32_t cmf = get(8), flg = get(8);
    if ((cmf & 15) != 8 || (cmf >> 4) > 7 || ((cmf << 8) | flg) % 31 != 0 || (flg & 0x20)) return fail(err);
    mode = kHeader;
  }

  __device__ void header(Smem& sm, int t, unsigned int* err) {
    if (consumed_bits() > csize * 8ull) return fail(err);  // ran past the stream
    refill();
    last = get(1);
    const uint32_t type = get(2);
    uint8_t lens[320];
    if (type == 0) {  // stored
      get(n & 7);
      refill();
      const uint32_t len = get(16), nlen = get(16);
      if (len != (~nlen & 0xFFFFu) || pos() + len > usize) return fail(err);
      rem = len;
      mode = kStored;
      return;
    }
    if (type == 3) return fail(err);
    if (type == 1) {  // fixed Huffman codes
      for (int i = 0; i < 144; ++i) lens[i] = 8;
      for (int i = 144; i < 256; ++i) lens[i] = 9;
      for (int i = 256; i < 280; ++i) lens[i] = 7;
      for (int i = 280; i < 288; ++i) lens[i] = 8;
      build_table(lens, 288, false, sm.lsym, sm.lbase, llim, t);
      for (int i = 0; i < 32; ++i) lens[i] = 5;
      build_table(lens, 32, false, sm.dsym, sm.dbase, dlim, t);
      mode = kSym;
      return;
    }
    // dynamic Huffman codes
    refill();
    const int hlit = static_cast<int>(get(5)) + 257, hdist = static_cast<int>(get(5)) + 1,
              hclen = static_cast<int>(get(4)) + 4;
    if (hlit > 286 || hdist > 30) return fail(err);
    for (int i = 0; i < 19; ++i) lens[i] = 0;
    for (int i = 0; i < hclen; ++i) {
      refill();
      lens[c_clorder[i]] = static_cast<uint8_t>(get(3));
    }
    // the code-length code goes into the distance slots; the real distance code overwrites it
    if (!build_table(lens, 19, true, sm.dsym, sm.dbase, dlim, t)) return fail(err);
    const int total = hlit + hdist;
    int i = 0;
    while (i < total) {
      refill();
      const int s = decode(dlim, sm.dsym, sm.dbase, t);
      if (s < 0) return fail(err);
      if (s < 16) {
        lens[i++] = static_cast<uint8_t>(s);
        continue;
      }
      uint8_t v = 0;
      int rep;
      if (s == 16) {
        if (i == 0) return fail(err);
        v = lens[i - 1];
        rep = 3 + static_cast<int>(get(2));
      } else if (s == 17) {
        rep = 3 + static_cast<int>(get(3));
      } else {
        rep = 11 + static_cast<int>(get(7));
      }
      if (i + rep > total) return fail(err);
      while (rep--) lens[i++] = v;
    }
    if (lens[256] == 0) return fail(err);  // no end-of-block code
    if (!build_table(lens, hlit, false, sm.lsym, sm.lbase, llim, t)) return fail(err);
    if (!build_table(lens + hlit, hdist, false, sm.dsym, sm.dbase, dlim, t)) return fail(err);
    mode = kSym;
  }

  __device__ void trailer(unsigned int* err) {
    get(n & 7);  // byte align
    refill();
    const uint32_t want = __byte_perm(get(32), 0, 0x0123);  // Adler-32 is big-endian
    if (consumed_bits() > csize * 8ull || pos() != usize) return fail(err);
    uint32_t a = s1 % 65521u, c = s2 % 65521u;
    for (int k = 0; k < an; ++k) {  // sizes that are not a multiple of 8 (never for column chunks)
      const uint32_t byte = static_cast<uint32_t>(acc >> (8 * k)) & 0xFFu;
      reinterpret_cast<uint8_t*>(dst)[oi + k] = static_cast<uint8_t>(byte);
      a = (a + byte) % 65521u;
      c = (c + a) % 65521u;
    }
    if (want != ((c << 16) | a)) return fail(err);
    j += stride;
    mode = kStart;
  }
};

__global__ void __launch_bounds__(kThreads) k_inflate(const InflateJob* __restrict__ jobs, uint32_t njobs,
                                                     unsigned int* err) {
  __shared__ Smem sm;
  const int t = threadIdx.x;
  Lane L;
  L.jobs = jobs;
  L.njobs = njobs;
  L.j = blockIdx.x * kThreads + t;
  L.stride = gridDim.x * kThreads;
  L.mode = kStart;
#pragma unroll
  for (int l = 0; l < 16; ++l) L.llim[l] = L.dlim[l] = 0;
  while (__any_sync(0xFFFFFFFFu, L.mode != kIdle)) {
    if (L.mode == kSym) {
      L.refill();
      int s = L.decode(L.llim, sm.lsym, sm.lbase, t);
      if (s < 0) {
        L.fail(err);
      } else if (s < 256) {
        if (L.pos() >= L.usize) {
          L.fail(err);
        } else {
          L.put(static_cast<uint64_t>(s), 1);
        }
      } else if (s == 256) {
        L.mode = L.last ? kTrailer : kHeader;
      } else if (s - 257 >= 29) {
        L.fail(err);
      } else {
        s -= 257;
        const uint32_t len = c_lbase[s] + L.get(c_lext[s]);
        L.refill();
        const int ds = L.decode(L.dlim, sm.dsym, sm.dbase, t);
        if (ds < 0 || ds >= 30) {
          L.fail(err);
        } else {
          const uint32_t dist = c_dbase[ds] + L.get(c_dext[ds]);
          const uint64_t q = L.pos();
          if (dist > q || q + len > L.usize) {
            L.fail(err);
          } else {
            L.rem = len;
            L.dist = dist;
            L.mode = kCopy;
          }
        }
      }
    } else if (L.mode == kCopy) {
      const int k = L.rem < 8 ? static_cast<int>(L.rem) : 8;
      uint64_t v;
      if (L.dist >= 8) {
        v = L.read8(L.pos() - L.dist);
      } else {  // period < 8: replicate the last `dist` bytes
        const int d = static_cast<int>(L.dist);
        v = low_bytes(L.last8() >> (8 * (8 - d)), d);
        v |= shl(v, 8 * d);
        v |= shl(v, 16 * d);
        v |= shl(v, 32 * d);
      }
      L.put(v, k);
      L.rem -= k;
      if (L.rem == 0) L.mode = kSym;
    } else if (L.mode == kStored) {
      if (L.rem == 0) {
        L.mode = L.last ? kTrailer : kHeader;
      } else {
        const int k = L.rem < 4 ? static_cast<int>(L.rem) : 4;
        L.refill();
        L.put(L.get(8 * k), k);
        L.rem -= k;
      }
    } else if (L.mode == kHeader) {
      L.header(sm, t, err);
    } else if (L.mode == kTrailer) {
      L.trailer(err);
    } else if (L.mode == kStart) {
      L.start(err);
    }
  }
}

}  // namespace

void launch_inflate(const InflateJob* d_jobs, uint32_t njobs, unsigned int* d_err, void* stream) {
  if (njobs == 0) return;
  // persistent lanes: each takes jobs j, j + stride, ... (longest first, see plan_batches)
  const uint32_t blocks = std::min<uint32_t>((njobs + kThreads - 1) / kThreads, 148u * 4u);
  k_inflate<<<blocks, kThreads, 0, static_cast<cudaStream_t>(stream)>>>(d_jobs, njobs, d_err);
  count_external_launch();
}

}  // namespace psg
