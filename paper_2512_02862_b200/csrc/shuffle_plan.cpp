#include "shuffle_plan.hpp"

#include "common.hpp"

namespace psg {

ExchangePlan plan_exchange(const uint64_t* m, int n, int me) {
  if (n < 1 || me < 0 || me >= n) throw InvalidInput("exchange plan: rank out of range");
  ExchangePlan x;
  x.send_cnt.resize(n);
  x.send_off.resize(n);
  x.recv_cnt.resize(n);
  x.recv_off.resize(n);
  for (int p = 0; p < n; ++p) {
    x.send_cnt[p] = m[static_cast<size_t>(me) * n + p];
    x.recv_cnt[p] = m[static_cast<size_t>(p) * n + me];
    x.send_off[p] = x.send_rows;
    x.recv_off[p] = x.recv_rows;
    x.send_rows += x.send_cnt[p];
    x.recv_rows += x.recv_cnt[p];
  }
  return x;
}

PackLayout plan_pack(const int64_t* lo, const int64_t* hi, int ncols) {
  PackLayout L;
  L.fits = ncols > 1;
  for (int k = 0; k < ncols; ++k) {
    L.min.push_back(0);
    L.shift.push_back(L.bits);
    L.mask.push_back(0);
    if (hi[k] < lo[k]) {  // no rows anywhere: an empty field (but the key must be a real one)
      if (k == 0) L.fits = false;
      continue;
    }
    const uint64_t span = static_cast<uint64_t>(hi[k]) - static_cast<uint64_t>(lo[k]);
    const int w = span ? 64 - __builtin_clzll(span) : 0;
    if (L.bits + w > 64 || (k == 0 && w == 0)) L.fits = false;
    L.min[k] = lo[k];
    L.mask[k] = w == 64 ? ~0ULL : ((1ULL << w) - 1);
    L.bits += w;
  }
  return L;
}

}  // namespace psg
