// GPU inflate for the PSTO block codec (zlib streams, deflate level 1 at write time).
//
// The reference decodes every compressed column chunk on the host with zlib's uncompress
// (codec_decompress, psto.cpp:133-143, called per chunk from decode_group, scan.cpp:139-160) and
// raises IoFailure("inflate failed") on any error or size mismatch. Here the compressed chunks
// travel host->HBM as they are (3-8x fewer PCIe bytes than decoded columns) and are expanded in
// HBM by this kernel, straight into the chunk layout the fused scan kernel reads.
//
// Design (B200): one warp per chunk (persistent warps walk the job list, longest first).
//   * Huffman decoding is inherently serial, so the whole warp runs it in lockstep on identical
//     state (a warp instruction costs one issue slot however many lanes are active), with one
//     shared-memory lookup per symbol: 10-bit (literal/length) and 8-bit (distance) first-level
//     tables whose entries carry code length, kind, literal / base length / base distance and
//     extra-bit count; the rare longer codes fall back to canonical decoding (left-justified
//     per-length limits held in registers).
//   * Output goes to a 2 KB per-warp ring that always holds the last 2 KB. A literal is one byte
//     store; a match is copied by the 32 lanes at once (lane i writes byte pos + i from byte
//     pos - dist + i mod dist, one round per 32 bytes), so its cost does not grow with its length
//     up to 32 bytes. Sources older than the ring come from the already flushed output in HBM.
//   * Parallel parts: table construction (histogram by warp reduction, canonical symbol order by
//     match masks, each lane fills 32 of the 1024 table slots), stored-block copies (32 bytes per
//     round) and the flush of every 1 KB of output as coalesced 16-byte stores, with the Adler-32
//     of the flushed bytes folded in by a dp4a warp reduction (zlib verifies the trailer; so do we).
// Every failure zlib reports (bad header, reserved block type, over-subscribed or incomplete
// codes, invalid symbols, distance too far back, output overrun or short output, reading past the
// stream, Adler mismatch) sets the error word; the host raises IoFailure("inflate failed").
#include <algorithm>
#include <cstdint>

#include "kernels.cuh"

namespace psg {
namespace {

constexpr int kWarps = 4;                  // warps (= concurrent chunks) per CTA
constexpr int kLB = 10, kDB = 8, kCB = 7;  // first-level table bits: lit/len, distance, code-length
constexpr uint32_t kRing = 2048, kRingMask = kRing - 1;
constexpr uint32_t kFlush = 1024;             // output flushed to HBM in 1 KB pieces
constexpr uint32_t kFull = 0xFFFFFFFFu;

__constant__ uint16_t c_lbase[29] = {3,  4,  5,  6,  7,  8,  9,  10, 11,  13,  15,  17,  19,  23, 27,
                                     31, 35, 43, 51, 59, 67, 83, 99, 115, 131, 163, 195, 227, 258};
__constant__ uint8_t c_lext[29] = {0, 0, 0, 0, 0, 0, 0, 0, 1, 1, 1, 1, 2, 2, 2, 2, 3, 3, 3, 3, 4, 4, 4, 4, 5, 5, 5, 5, 0};
__constant__ uint16_t c_dbase[30] = {1,   2,   3,   4,   5,   7,    9,    13,   17,   25,   33,   49,   65,    97,    129,
                                     193, 257, 385, 513, 769, 1025, 1537, 2049, 3073, 4097, 6145, 8193, 12289, 16385, 24577};
__constant__ uint8_t c_dext[30] = {0, 0, 0, 0, 1, 1, 2, 2, 3, 3, 4, 4, 5, 5, 6, 6, 7, 7, 8, 8, 9, 9, 10, 10, 11, 11, 12, 12, 13, 13};
__constant__ uint8_t c_clorder[19] = {16, 17, 18, 0, 8, 7, 9, 6, 10, 5, 11, 4, 12, 3, 13, 2, 14, 1, 15};

// First-level table entries. Literal/length (16 bits): bits 0-3 code length (0 = longer than the
// table: decode canonically), bit 4 literal flag; a literal keeps its byte in bits 8-15, any other
// symbol keeps in bits 5-7 its extra-bit count (0-5 for a length; 6 end of block; 7 invalid or long
// code) and in bits 8-15 its base length - 3. Distance / code-length (32 bits): bits 0-3 code
// length, bit 4 slow flag (invalid, or longer than the table), bits 8-11 extra-bit count, bits
// 16-31 base distance or code-length symbol.
constexpr uint32_t kLitFlag = 0x10u, kSlow = 0x10u;
constexpr uint32_t kXEob = 6u, kXSlow = 7u;
constexpr uint32_t kBadEntry = kSlow | 1u;  // bits that match no code

struct alignas(16) WarpSmem {
  uint8_t ring[kRing];
  uint16_t lfast[1 << kLB];
  uint32_t dfast[1 << kDB];  // also the code-length table (kCB bits) while reading a header
  uint16_t lsym[288];
  uint16_t dsym[32];
  int32_t lbase[16];
  int32_t dbase[16];
  uint32_t llim[16];  // left-justified per-length limits of the canonical codes
  uint32_t dlim[16];
  uint8_t lens[320];
};
static_assert(sizeof(WarpSmem) * kWarps <= 26 * 1024, "inflate shared memory: 8 CTAs per SM");

/// Canonical Huffman decode of the next code (lane 0): -1 when the bits match no code.
__device__ __forceinline__ int canon_decode(uint64_t bits, const uint32_t* lim, const int32_t* base,
                                            const uint16_t* sym, int& len) {
  const uint32_t c15 = __brev(static_cast<uint32_t>(bits)) >> 17;
  len = 1;
#pragma unroll
  for (int l = 1; l < 16; ++l) len += (c15 >= lim[l]) ? 1 : 0;
  if (len > 15) return -1;
  return sym[base[len] + static_cast<int>(c15 >> (15 - len))];
}

/// Builds a canonical code from lens[0, n) into sym/base/lim (shared) and fills the first-level
/// table `fast` (2^fb entries; 16-bit entries for literal/length) cooperatively. `what`: 0 literal/length,
/// 1 distance, 2 code-length code. Returns false (in all lanes) for codes zlib rejects
/// (inflate_table: over-subscribed, or incomplete unless a single one-bit lit/len or distance code).
__device__ bool build_table(const uint8_t* lens, int n, int what, uint16_t* sym, int32_t* base, void* fast_, int fb,
                            uint32_t* slim, int lane) {
  uint32_t lim[16];
  uint32_t cnt[16];
#pragma unroll
  for (int l = 0; l < 16; ++l) cnt[l] = 0;
  for (int i = lane; i < n; i += 32) {  // each lane histograms a slice ...
    const int l = lens[i];
#pragma unroll
    for (int k = 1; k < 16; ++k) cnt[k] += (l == k) ? 1u : 0u;
  }
#pragma unroll
  for (int k = 1; k < 16; ++k) cnt[k] = __reduce_add_sync(kFull, cnt[k]);  // ... then one reduction per length
  int maxlen = 0, left = 1;
  bool ok = true;
#pragma unroll
  for (int l = 1; l < 16; ++l) {
    if (cnt[l]) maxlen = l;
    left = (left << 1) - static_cast<int>(cnt[l]);
    if (left < 0) ok = false;  // over-subscribed
  }
  if (ok && maxlen > 0 && left > 0 && (what == 2 || maxlen != 1)) ok = false;  // incomplete
  if (!ok) return false;
  uint32_t offs[16];
  uint32_t code = 0, off = 0;
#pragma unroll
  for (int l = 1; l < 16; ++l) {
    offs[l] = off;
    lim[l] = (code + cnt[l]) << (15 - l);
    if (lane == 0) base[l] = static_cast<int32_t>(off) - static_cast<int32_t>(code);
    if (lane == 0) slim[l] = lim[l];
    code = (code + cnt[l]) << 1;
    off += cnt[l];
  }
  // symbols in canonical order, 32 at a time: rank within a length from the match mask
  for (int g = 0; g < n; g += 32) {
    const int i = g + lane;
    const int l = i < n ? lens[i] : 0;
    const uint32_t same = __match_any_sync(kFull, l);
    const uint32_t rank = __popc(same & ((1u << lane) - 1u));
    uint32_t my_off = 0;
#pragma unroll
    for (int k = 1; k < 16; ++k) {
      if (l == k) my_off = offs[k];
      offs[k] += __popc(__ballot_sync(kFull, l == k));
    }
    if (l) sym[my_off + rank] = static_cast<uint16_t>(i);
  }
  __syncwarp();
  // first-level table: slot e holds the decode of bit pattern e (stream order, LSB first)
  const int slots = 1 << fb;
  for (int e = lane; e < slots; e += 32) {
    const uint32_t c15 = (__brev(static_cast<uint32_t>(e)) >> (32 - fb)) << (15 - fb);
    int len = 1;
#pragma unroll
    for (int l = 1; l < 16; ++l) len += (c15 >= lim[l]) ? 1 : 0;
    uint32_t ent;
    if (len > 15) {
      ent = what == 0 ? ((kXSlow << 5) | 1u) : kBadEntry;
    } else if (len > fb) {
      ent = what == 0 ? (kXSlow << 5) : kSlow;  // code length 0: decode canonically
    } else {
      const int s = sym[base[len] + static_cast<int>(c15 >> (15 - len))];
      const uint32_t L = static_cast<uint32_t>(len);
      if (what == 0) {
        if (s < 256) ent = L | kLitFlag | (static_cast<uint32_t>(s) << 8);
        else if (s == 256) ent = L | (kXEob << 5);
        else if (s < 286) ent = L | (static_cast<uint32_t>(c_lext[s - 257]) << 5) |
                                (static_cast<uint32_t>(c_lbase[s - 257] - 3) << 8);
        else ent = L | (kXSlow << 5);  // symbols 286, 287: invalid
      } else if (what == 1) {
        ent = s < 30 ? L | (static_cast<uint32_t>(c_dext[s]) << 8) | (static_cast<uint32_t>(c_dbase[s]) << 16)
                     : L | kSlow;
      } else {
        ent = L | (static_cast<uint32_t>(s) << 16);
      }
    }
    if (what == 0) static_cast<uint16_t*>(fast_)[e] = static_cast<uint16_t>(ent);
    else static_cast<uint32_t*>(fast_)[e] = ent;
  }
  __syncwarp();
  return true;
}

/// Bit reader: LSB-first over 4-byte aligned words (chunks are 16-byte aligned). Every lane of
/// the warp holds the same state (the loads are broadcasts).
struct Bits {
  const uint32_t* w0;  // stream start
  uint32_t nlast;      // last word that may be loaded (chunks are padded to 16 bytes)
  uint32_t next;       // index of the word in `nw`
  uint32_t nw;         // prefetched next word: its load is off the decode chain
  uint64_t b;
  int n;
  __device__ __forceinline__ void start(const void* src, uint32_t csize) {
    w0 = reinterpret_cast<const uint32_t*>(src);
    nlast = csize > 4 ? (csize - 1) / 4 : 0;
    next = 0;
    nw = __ldg(w0);
    b = 0;
    n = 0;
  }
  // Past the stream the reader feeds repeats of the last word; any stream that consumes them is
  // rejected by the consumed-bits checks (block headers, trailer), as zlib rejects it.
  __device__ __forceinline__ void refill() {
    if (n <= 32) {
      b |= static_cast<uint64_t>(nw) << n;
      n += 32;
      ++next;
      nw = __ldg(w0 + min(next, nlast));
    }
  }
  /// Appends the prefetched word (n <= 32).
  __device__ __forceinline__ void refill_now() {
    __syncwarp();  // (also keeps the rare call sites branches rather than predicated code)
    b |= static_cast<uint64_t>(nw) << n;
    n += 32;
    ++next;
    nw = __ldg(w0 + min(next, nlast));
  }
  __device__ __forceinline__ uint32_t get(int k) {  // k <= 32, n >= k
    const uint32_t v = static_cast<uint32_t>(b & ((1ull << k) - 1ull));
    b >>= k;
    n -= k;
    return v;
  }
  __device__ __forceinline__ void drop(int k) {
    b >>= k;
    n -= k;
  }
  /// Drops a k-bit code and returns the x extra bits after it (k + x <= 32, n >= k + x).
  __device__ __forceinline__ uint32_t code_extra(int k, int x) {
    const uint32_t v = (static_cast<uint32_t>(b) >> k) & ((1u << x) - 1u);
    b >>= k + x;
    n -= k + x;
    return v;
  }
  __device__ __forceinline__ uint64_t consumed() const { return static_cast<uint64_t>(next) * 32ull - n; }
  __device__ __forceinline__ void seek(uint64_t bit) {  // restart at an absolute bit position
    next = static_cast<uint32_t>(bit >> 5);
    nw = __ldg(w0 + min(next, nlast));
    b = 0;
    n = 0;
    refill();
    drop(static_cast<int>(bit & 31));
  }
};

// decode-section outcomes
enum Reason : int { kRFlush = 0, kREob = 1, kRErr = 2 };

/// Output state (identical in every lane): `pos` bytes produced; the ring holds the last 2 KB.
struct Out {
  uint8_t* ring;
  const uint8_t* hbm;  // the chunk's output, flushed up to the warp's `flushed`
  uint32_t pos;
  /// One literal byte.
  __device__ __forceinline__ void lit(uint32_t byte) {
    ring[pos & kRingMask] = static_cast<uint8_t>(byte);
    ++pos;
  }
  /// A match, copied by the whole warp 32 bytes per round. Output byte pos + i repeats byte
  /// pos - dist + (i mod dist), which always precedes pos, so the rounds are independent: every
  /// source is read before the round's stores, and a store only recycles the ring slot of a byte
  /// 2 KB back. Sources within 2 KB come from the ring, older ones from the flushed output (at
  /// least 1790 bytes back, while the flush trails pos by less than 1282).
  __device__ __forceinline__ void match(uint32_t len, uint32_t dist, int lane) {
    const uint32_t s0 = pos - dist;
    const bool wrap = dist < len;  // the period repeats inside the match
    const float rd = wrap ? __frcp_rn(static_cast<float>(dist)) : 0.f;
    const bool near = dist <= kRing;
    auto copy = [&](uint32_t i) {
      if (i < len) {
        uint32_t off = i;
        if (wrap) {  // i mod dist: (i + 1/2) / dist is >= 1/(2 dist) away from an integer
          const uint32_t q = static_cast<uint32_t>((static_cast<float>(i) + 0.5f) * rd);
          off = i - q * dist;
        }
        const uint32_t src = s0 + off;
        const uint8_t v = near ? ring[src & kRingMask] : __ldcg(hbm + src);
        ring[(pos + i) & kRingMask] = v;
      }
    };
    copy(static_cast<uint32_t>(lane));
    if (len > 32) {
#pragma unroll 1
      for (uint32_t base = 32; base < len; base += 32) copy(base + static_cast<uint32_t>(lane));
    }
    __syncwarp();  // the copied bytes are sources / flush input for other lanes
    pos += len;
  }
};

/// Flushes ring bytes [flushed, flushed + nbytes) (nbytes <= kFlush) to dst in whole 16-byte
/// granules (chunk buffers are padded to 16 bytes) and folds them into the Adler-32 state
/// (s1, s2 identical in every lane).
__device__ __forceinline__ void flush(const uint8_t* ring, uint8_t* dst, uint32_t flushed, uint32_t nbytes, uint32_t& s1,
                                      uint32_t& s2, int lane) {
  const uint32_t mine = static_cast<uint32_t>(lane) * 32u;
  uint32_t A = 0, B = 0;
  if (mine < nbytes) {
    const uint32_t rp = (flushed + mine) & kRingMask;  // 32-byte aligned, never wraps
    const uint4 x = *reinterpret_cast<const uint4*>(ring + rp);
    const uint4 y = *reinterpret_cast<const uint4*>(ring + rp + 16);
    uint32_t w[8] = {x.x, x.y, x.z, x.w, y.x, y.y, y.z, y.w};
    const uint32_t valid = min(32u, nbytes - mine);
    if (valid < 32) {  // zero the bytes past the end of the stream
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int keep = static_cast<int>(valid) - 4 * k;
        w[k] = keep >= 4 ? w[k] : (keep <= 0 ? 0u : (w[k] & ((1u << (8 * keep)) - 1u)));
      }
    }
    uint4* d = reinterpret_cast<uint4*>(dst + flushed + mine);
    d[0] = make_uint4(w[0], w[1], w[2], w[3]);
    if (valid > 16) d[1] = make_uint4(w[4], w[5], w[6], w[7]);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      A = __dp4a(w[k], 0x01010101u, A);
      // weights 32 - m for bytes m = 4k..4k+3 of this lane's slice
      const uint32_t wt = (32u - 4u * k) | ((31u - 4u * k) << 8) | ((30u - 4u * k) << 16) | ((29u - 4u * k) << 24);
      B = __dp4a(w[k], wt, B);
    }
  }
  // a block of N bytes: s2 += N*s1 + sum_i [(N - 32i - 32) A_i + B_i], s1 += sum_i A_i
  const int32_t tail = static_cast<int32_t>(nbytes) - static_cast<int32_t>(mine) - 32;
  const uint32_t part = static_cast<uint32_t>(static_cast<int32_t>(B) + tail * static_cast<int32_t>(A));
  const uint32_t SA = __reduce_add_sync(kFull, A);
  const uint32_t SB = __reduce_add_sync(kFull, part);
  s2 = (s2 + nbytes * s1 + SB) % 65521u;
  s1 = (s1 + SA) % 65521u;
}

/// The warp's decode loop for one data phase (every lane runs it in lockstep): runs until 1 KB
/// is ready to flush, the block ends or the stream is invalid. Stored blocks (type 0) copy
/// `stored` more bytes; else Huffman symbols.
__device__ __forceinline__ int decode_run(Bits& br, Out& o, WarpSmem& sm, int type, uint32_t& stored, uint32_t flushed,
                                          uint32_t usize, uint32_t csize, int lane) {
  // Output past usize is caught here, before its flush could write outside the chunk (the ring
  // absorbs up to one match past the flush point), or by the trailer's exact-size check.
  const uint32_t limit = flushed + kFlush;
  if (type == 0) {  // byte aligned: the warp copies 32 stream bytes per round
    const uint64_t bit = br.consumed();
    const uint8_t* src = reinterpret_cast<const uint8_t*>(br.w0) + (bit >> 3);
    const uint32_t avail = csize > (bit >> 3) ? csize - static_cast<uint32_t>(bit >> 3) : 0u;
    uint32_t done = 0;
    int r = kREob;
    while (done < stored) {
      const uint32_t k = min(32u, stored - done);
      if (static_cast<uint32_t>(lane) < k) {
        const uint32_t j = done + static_cast<uint32_t>(lane);
        o.ring[(o.pos + static_cast<uint32_t>(lane)) & kRingMask] = j < avail ? __ldg(src + j) : 0;
      }
      o.pos += k;
      done += k;
      if (o.pos >= limit) {
        r = o.pos > usize ? kRErr : kRFlush;
        break;
      }
    }
    stored -= done;
    br.seek(bit + 8ull * done);
    return r;
  }
  while (true) {
    br.refill();
    uint32_t e = sm.lfast[br.b & ((1u << kLB) - 1u)];
    if (e & kLitFlag) {
      // Literals with short codes, the hot path: a refill leaves >= 33 bits, enough for three
      // 10-bit lookups; the flush check runs once per group (the ring has room past the limit).
      br.drop(static_cast<int>(e & 15));
      o.lit(e >> 8);
      e = sm.lfast[br.b & ((1u << kLB) - 1u)];
      if (e & kLitFlag) {
        br.drop(static_cast<int>(e & 15));
        o.lit(e >> 8);
        e = sm.lfast[br.b & ((1u << kLB) - 1u)];
        if (e & kLitFlag) {
          br.drop(static_cast<int>(e & 15));
          o.lit(e >> 8);
          if (o.pos >= limit) return o.pos > usize ? kRErr : kRFlush;
          continue;
        }
      }
      if (o.pos >= limit) return o.pos > usize ? kRErr : kRFlush;
      if (__builtin_expect(br.n < 15, 0)) br.refill_now();  // (>= 13 bits left) a length code + its extra bits; e stays valid
    }
    uint32_t x = (e >> 5) & 7, len;
    if (x < kXEob) {  // length with a short code
      len = (e >> 8) + 3 + br.code_extra(static_cast<int>(e & 15), static_cast<int>(x));
    } else {  // cold: end of block, invalid bits, or a code longer than the table
      int cl = static_cast<int>(e & 15);
      if (x == kXEob) {
        br.drop(cl);
        return kREob;
      }
      if (cl != 0) return kRErr;
      br.refill();  // a long code + extra bits: <= 20
      const int s = canon_decode(br.b, sm.llim, sm.lbase, sm.lsym, cl);
      if (s < 0 || s >= 286) return kRErr;
      br.drop(cl);
      if (s == 256) return kREob;
      if (s < 256) {
        o.lit(static_cast<uint32_t>(s));
        if (o.pos >= limit) return o.pos > usize ? kRErr : kRFlush;
        continue;
      }
      len = c_lbase[s - 257] + br.get(c_lext[s - 257]);
    }
    // the 8-bit lookup and a short distance code + its extra bits need <= 21 bits
    if (__builtin_expect(br.n < 21, 0)) br.refill_now();
    uint32_t de = sm.dfast[br.b & ((1u << kDB) - 1u)];
    int dl = static_cast<int>(de & 15);
    if (de & kSlow) {
      if (dl != 0) return kRErr;
      br.refill();  // a long code + extra bits: <= 28
      const int s = canon_decode(br.b, sm.dlim, sm.dbase, sm.dsym, dl);
      if (s < 0 || s >= 30) return kRErr;
      de = (static_cast<uint32_t>(c_dext[s]) << 8) | (static_cast<uint32_t>(c_dbase[s]) << 16);
    }
    const uint32_t dist = (de >> 16) + br.code_extra(dl, static_cast<int>((de >> 8) & 15));
    if (dist >= len && dist <= kRing && len <= 32 && dist <= o.pos) {
      // the common match: sources in the ring, no overlap with the output, one round
      if (static_cast<uint32_t>(lane) < len)
        o.ring[(o.pos + static_cast<uint32_t>(lane)) & kRingMask] = o.ring[(o.pos - dist + static_cast<uint32_t>(lane)) & kRingMask];
      __syncwarp();
      o.pos += len;
    } else {
      if (dist > o.pos) return kRErr;
      o.match(len, dist, lane);
    }
    if (o.pos >= limit) return o.pos > usize ? kRErr : kRFlush;
  }
}

__global__ void __launch_bounds__(kWarps * 32, 8) k_inflate(const InflateJob* __restrict__ jobs, uint32_t njobs,
                                                        unsigned int* err) {
  __shared__ WarpSmem smem[kWarps];
  const int lane = threadIdx.x & 31;
  WarpSmem& sm = smem[threadIdx.x >> 5];
  const uint32_t nwarps = gridDim.x * kWarps;

  for (uint32_t j = blockIdx.x * kWarps + (threadIdx.x >> 5); j < njobs; j += nwarps) {
    const InflateJob job = jobs[j];
    const uint32_t usize = job.usize;
    uint8_t* const dst = job.dst;
    Bits br;
    br.start(job.src, job.csize);
    Out o;
    o.ring = sm.ring;
    o.hbm = dst;
    o.pos = 0;
    uint32_t flushed = 0, s1 = 1, s2 = 0;
    bool ok, last = false;
    {  // zlib header (RFC 1950): deflate, window <= 32K, no preset dictionary, FCHECK
      br.refill();
      const uint32_t cmf = br.get(8), flg = br.get(8);
      ok = !((cmf & 15) != 8 || (cmf >> 4) > 7 || ((cmf << 8) | flg) % 31 != 0 || (flg & 0x20));
    }
    // Every lane runs the serial parts in lockstep on identical state (one issue slot either
    // way); shared-memory stores of those parts write one value to one address from all lanes.
    while (ok && !last) {
      // ---------------- block header, then the warp builds the tables
      if (br.consumed() > job.csize * 8ull) {  // ran past the stream
        ok = false;
        break;
      }
      br.refill();
      last = br.get(1) != 0;
      const int type = static_cast<int>(br.get(2));
      uint32_t stored = 0;
      if (type == 3) {
        ok = false;
        break;
      }
      if (type == 0) {
        br.drop(br.n & 7);
        br.refill();
        stored = br.get(16);
        const uint32_t nlen = br.get(16);
        if (stored != (~nlen & 0xFFFFu) || o.pos + stored > usize) {
          ok = false;
          break;
        }
      } else if (type == 1) {  // fixed codes
        for (int i = lane; i < 288; i += 32) sm.lens[i] = i < 144 ? 8 : (i < 256 ? 9 : (i < 280 ? 7 : 8));
        __syncwarp();
        build_table(sm.lens, 288, 0, sm.lsym, sm.lbase, sm.lfast, kLB, sm.llim, lane);
        sm.lens[lane] = 5;
        __syncwarp();
        build_table(sm.lens, 32, 1, sm.dsym, sm.dbase, sm.dfast, kDB, sm.dlim, lane);
      } else {  // dynamic codes: the code-length code, then both code-length sequences
        br.refill();
        const int hlit = static_cast<int>(br.get(5)) + 257;
        const int hdist = static_cast<int>(br.get(5)) + 1;
        const int hclen = static_cast<int>(br.get(4)) + 4;
        if (hlit > 286 || hdist > 30) {
          ok = false;
          break;
        }
        if (lane < 19) sm.lens[lane] = 0;
        __syncwarp();
        for (int i = 0; i < hclen; ++i) {
          br.refill();
          sm.lens[c_clorder[i]] = static_cast<uint8_t>(br.get(3));
        }
        __syncwarp();
        if (!build_table(sm.lens, 19, 2, sm.dsym, sm.dbase, sm.dfast, kCB, sm.dlim, lane)) {
          ok = false;
          break;
        }
        const int total = hlit + hdist;
        int i = 0;
        bool bad = false;
        uint8_t prev = 0;
        while (i < total) {
          br.refill();
          const uint32_t e = sm.dfast[br.b & ((1u << kCB) - 1u)];
          if (e & kSlow) {  // bits outside the code-length code
            bad = true;
            break;
          }
          br.drop(static_cast<int>(e & 15));
          const int sy = static_cast<int>(e >> 16);
          if (sy < 16) {
            sm.lens[i++] = prev = static_cast<uint8_t>(sy);
            continue;
          }
          uint8_t v = 0;
          int rep;
          if (sy == 16) {
            if (i == 0) {
              bad = true;
              break;
            }
            v = prev;
            rep = 3 + static_cast<int>(br.get(2));
          } else if (sy == 17) {
            rep = 3 + static_cast<int>(br.get(3));
          } else {
            rep = 11 + static_cast<int>(br.get(7));
          }
          if (i + rep > total) {
            bad = true;
            break;
          }
          if (lane < rep) sm.lens[i + lane] = v;  // rep <= 138: at most 5 rounds
          if (lane + 32 < rep) sm.lens[i + lane + 32] = v;
          if (lane + 64 < rep) sm.lens[i + lane + 64] = v;
          if (lane + 96 < rep) sm.lens[i + lane + 96] = v;
          if (lane + 128 < rep) sm.lens[i + lane + 128] = v;
          i += rep;
          prev = v;
        }
        __syncwarp();
        if (bad || sm.lens[256] == 0) {  // (no end-of-block code)
          ok = false;
          break;
        }
        if (!build_table(sm.lens, hlit, 0, sm.lsym, sm.lbase, sm.lfast, kLB, sm.llim, lane) ||
            !build_table(sm.lens + hlit, hdist, 1, sm.dsym, sm.dbase, sm.dfast, kDB, sm.dlim, lane)) {
          ok = false;
          break;
        }
      }
      // ---------------- data: the warp decodes; each finished 1 KB is flushed
      while (true) {
        const int reason = decode_run(br, o, sm, type, stored, flushed, usize, job.csize, lane);
        if (reason == kRErr) {
          ok = false;
          break;
        }
        __syncwarp();
        while (o.pos - flushed >= kFlush) {
          flush(sm.ring, dst, flushed, kFlush, s1, s2, lane);
          flushed += kFlush;
        }
        __syncwarp();
        if (reason == kREob) break;
      }
    }
    if (ok) {
      // ---------------- trailer: final flush, exact size, Adler-32
      const uint32_t P = o.pos;
      if (P != usize) ok = false;
      __syncwarp();
      if (ok && P > flushed) flush(sm.ring, dst, flushed, P - flushed, s1, s2, lane);
      if (ok) {
        br.drop(br.n & 7);
        br.refill();
        const uint32_t want = __byte_perm(br.get(32), 0, 0x0123);  // big-endian
        if (br.consumed() > job.csize * 8ull || want != ((s2 << 16) | s1)) ok = false;
      }
    }
    if (!ok && lane == 0) atomicOr(err, 1u);
    __syncwarp();
  }
}

}  // namespace

void launch_inflate(const InflateJob* d_jobs, uint32_t njobs, unsigned int* d_err, void* stream) {
  if (njobs == 0) return;
  // persistent warps: warp w takes jobs w, w + nwarps, ... (longest first, see plan_batches);
  // 8 CTAs x 4 warps fit an SM (25 KB of tables + ring per CTA, <= 64 registers)
  static bool attr = [] {
    return cudaFuncSetAttribute(k_inflate, cudaFuncAttributePreferredSharedMemoryCarveout,
                                cudaSharedmemCarveoutMaxShared) == cudaSuccess;
  }();
  (void)attr;
  const uint32_t blocks = std::min<uint32_t>((njobs + kWarps - 1) / kWarps, 148u * 8u);
  k_inflate<<<blocks, kWarps * 32, 0, static_cast<cudaStream_t>(stream)>>>(d_jobs, njobs, d_err);
  count_external_launch();
}

}  // namespace psg
