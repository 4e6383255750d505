using namespace psg;
#define R 4
extern "C" __global__ void __launch_bounds__(544, 2) psg_jit_scan(const __grid_constant__ ScanProgram P, const Segment* __restrict__ segs, const uint32_t* __restrict__ tile_seg, uint64_t ntiles) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* stg = reinterpret_cast<uint64_t*>(smem_raw);  // [4][2][1024]
  __shared__ __align__(8) uint64_t full_bar[4], empty_bar[4];
  __shared__ const uint64_t* s_col[4][4];
  __shared__ int s_rows[4];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int i = 0; i < 4; ++i) { mbar_init(&full_bar[i], 1); mbar_init(&empty_bar[i], 8); }
    mbar_fence_init();
  }
  __syncthreads();
  const uint64_t per_cta = (ntiles + gridDim.x - 1) / gridDim.x;
  const uint64_t t_beg = blockIdx.x * per_cta;
  const uint64_t t_end = t_beg + per_cta < ntiles ? t_beg + per_cta : ntiles;
  if (warp == 0) {  // producer
    if (lane == 0) {
      const uint64_t pol_stream = l2_evict_first();
      for (uint64_t k = 0; t_beg + k < t_end; ++k) {
        const int st = static_cast<int>(k % 4); const uint32_t ph = static_cast<uint32_t>((k / 4) & 1);
        if (k >= 4) mbar_wait(&empty_bar[st], ph ^ 1u);
        const uint64_t t = t_beg + k;
        const Segment* sg = segs + __ldg(tile_seg + t);
        const uint64_t r0 = (t - sg->tile_begin) * 1024ULL;
        const int rows = static_cast<int>(min(1024ULL, sg->rows - r0));
        s_col[st][2] = sg->col[2] + r0;
        s_col[st][3] = sg->col[3] + r0;
        s_rows[st] = rows;
        const uint32_t bytes = (static_cast<uint32_t>(rows) * 8u + 15u) & ~15u;
        mbar_arrive_expect_tx(&full_bar[st], 2u * bytes);
        bulk_g2s(stg + (st * 2 + 0) * 1024, sg->col[0] + r0, bytes, &full_bar[st], pol_stream);
        bulk_g2s(stg + (st * 2 + 1) * 1024, sg->col[1] + r0, bytes, &full_bar[st], pol_stream);
      }
    }
    return;
  }
  const uint64_t pol_keep = l2_evict_last(); (void)pol_keep;
  const int cw = (warp - 1) % 8, grp = (warp - 1) / 8;
  const int wrow = cw * (R * 32) + lane;
  for (uint64_t k = grp; t_beg + k < t_end; k += 2) {
    const int st = static_cast<int>(k % 4); const uint32_t ph = static_cast<uint32_t>((k / 4) & 1);
    mbar_wait(&full_bar[st], ph);
    const int nrows = s_rows[st] - cw * (R * 32);
    uint32_t pass = 0;
#pragma unroll
    for (int r = 0; r < R; ++r) if (r * 32 + lane < nrows) pass |= 1u << r;
    uint64_t v0[R] = {};
    uint64_t v1[R] = {};
    uint64_t v2[R] = {};
    uint64_t v3[R] = {};
#pragma unroll
    for (int r = 0; r < R; ++r) if (pass & (1u << r)) v0[r] = stg[(st * 2 + 0) * 1024 + wrow + r * 32];
#pragma unroll
    for (int r = 0; r < R; ++r) if (pass & (1u << r)) v1[r] = stg[(st * 2 + 1) * 1024 + wrow + r * 32];
    const uint64_t* lc2 = s_col[st][2];
    const uint64_t* lc3 = s_col[st][3];
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty_bar[st]);  // stage consumed: the producer may refill it
    { const long long lit = static_cast<long long>(P.atoms[0].lit);
#pragma unroll
      for (int r = 0; r < R; ++r) if (!(static_cast<long long>(v0[r]) > lit)) pass &= ~(1u << r);
    }
    { const AggTableDev& T = P.agg; uint32_t gw[R], bb[R], kr[R], sl[R]; unsigned long long kw[R]; uint32_t sel = 0;
#pragma unroll
      for (int r = 0; r < R; ++r) { const uint64_t key = v1[r];
        const uint64_t d = key - static_cast<uint64_t>(T.kmin);
        const bool ok = ((pass >> r) & 1u) && key != kEmptyKey && d < T.krange;
        bb[r] = static_cast<uint32_t>(d & 31); gw[r] = ok ? ldg_keep_u32(T.kbits + (d >> 5), pol_keep) : 0u; }
#pragma unroll
      for (int r = 0; r < R; ++r) if ((gw[r] >> bb[r]) & 1u) sel |= 1u << r;
#pragma unroll
      for (int r = 0; r < R; ++r) { kw[r] = 0; kr[r] = 0; if ((sel >> r) & 1u) {
        const uint64_t d = v1[r] - static_cast<uint64_t>(T.kmin);
        uint64_t a, b; ldg_keep_v2u64(T.krec + 2 * (d >> 6), pol_keep, a, b); kw[r] = a; kr[r] = static_cast<uint32_t>(b); } }
      pass = sel;
#pragma unroll
      for (int r = 0; r < R; ++r) if (pass & (1u << r)) v2[r] = __ldcs(reinterpret_cast<const unsigned long long*>(lc2 + wrow + r * 32));
#pragma unroll
      for (int r = 0; r < R; ++r) if (pass & (1u << r)) v3[r] = __ldcs(reinterpret_cast<const unsigned long long*>(lc3 + wrow + r * 32));
#pragma unroll
      for (int r = 0; r < R; ++r) { const uint32_t d6 = static_cast<uint32_t>((v1[r] - static_cast<uint64_t>(T.kmin)) & 63);
        sl[r] = kr[r] + static_cast<uint32_t>(__popcll(kw[r] & ((1ULL << d6) - 1ULL))); }
      { uint64_t ab[R]; unsigned apos[R];
#pragma unroll
      for (int r = 0; r < R; ++r) { ab[r] = 0; apos[r] = 0; if (!(pass & (1u << r))) continue;
        ab[r] = ((sl[r] >> 11) << P.bkt_sub_bits) | (threadIdx.x & ((1u << P.bkt_sub_bits) - 1u));
        apos[r] = atomicAdd(P.bkt_fill + ab[r], 1u); }
#pragma unroll
      for (int r = 0; r < R; ++r) { if (!(pass & (1u << r))) continue;
        uint64_t e = sl[r] & 2047ULL;
        e |= ((v2[r] - static_cast<uint64_t>(P.bkt_min[0])) & P.bkt_mask[0]) << P.bkt_shift[0];
        e |= ((v3[r] - static_cast<uint64_t>(P.bkt_min[1])) & P.bkt_mask[1]) << P.bkt_shift[1];
        if (apos[r] < P.bkt_cap) {
          P.bkt[ab[r] * P.bkt_cap + apos[r]] = e;
        } else {  // bucket full: the overflow list
          const unsigned o = atomicAdd(P.bkt_ovf_count, 1u);
          if (o < P.bkt_ovf_cap) { P.bkt_ovf[2 * o] = sl[r]; P.bkt_ovf[2 * o + 1] = e; }
        }
      } }
    }
  }
}
