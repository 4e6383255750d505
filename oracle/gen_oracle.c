/*
 * ORACLE — test infrastructure only. Nothing in the product path may link, import or execute this.
 * (Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg use oracle/.)
 *
 * Plain-C restatement of the reference's deterministic TPC-H-analog generator and PSTO writer,
 * used as an independent checker for the product generator and as the oracle's data source.
 *
 *   mt19937_64                 — the C++ <random> engine the reference uses (published algorithm:
 *                                Matsumoto & Nishimura 2000, 64-bit variant; std::mt19937_64
 *                                parameters n=312 m=156 r=31 a=0xB5026F5AA96619E9 ...).
 *   gen_customer/orders/lineitem — /root/reference/proj/src/workload.cpp:89-153
 *                                (seed = seed*0x9E3779B97F4A7C15 + {11,12,13}; the date expression
 *                                at :118-119 / :145-146 calls rng() three times inside one '+'
 *                                expression; GCC 13.3 -O2 evaluates them left-to-right (year, month,
 *                                day). This is pinned by byte-identical file hashes against the
 *                                reference generator in tests/golden/gen_hashes.json.)
 *   slice_for_node             — workload.cpp:73-87 (rows r ≡ node mod nodes)
 *   write_sharded/replicated   — /root/reference/proj/src/bench.cpp:48-81 (file placement dev(i%devices))
 *   TableWriter / encode_footer — /root/reference/proj/src/psto.cpp:144-229, :192-213
 *                                (row_group_rows = max(1, rg_bytes / (ncols*8)), :157-160)
 *   codec_compress             — psto.cpp:119-131 (zlib compress2 level 1 for the block codec)
 *
 * Build: oracle/Makefile -> oracle/_build/liboracle_gen.so (ctypes).
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <sys/stat.h>
#include <errno.h>
#include <zlib.h>

/* ---------------- mt19937_64 ---------------- */
#define MT_N 312
#define MT_M 156
typedef struct { uint64_t mt[MT_N]; int idx; } mt64;

static void mt_seed(mt64 *s, uint64_t seed) {
  s->mt[0] = seed;
  for (int i = 1; i < MT_N; ++i)
    s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
  s->idx = MT_N;
}

static uint64_t mt_next(mt64 *s) {
  if (s->idx >= MT_N) {
    const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL, A = 0xB5026F5AA96619E9ULL;
    for (int i = 0; i < MT_N; ++i) {
      uint64_t x = (s->mt[i] & UM) | (s->mt[(i + 1) % MT_N] & LM);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= A;
      s->mt[i] = s->mt[(i + MT_M) % MT_N] ^ xa;
    }
    s->idx = 0;
  }
  uint64_t y = s->mt[s->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

uint64_t orc_mt64_first(uint64_t seed, uint64_t skip) {
  mt64 s;
  mt_seed(&s, seed);
  for (uint64_t i = 0; i < skip; ++i) mt_next(&s);
  return mt_next(&s);
}

/* yyyymmdd with GCC's left-to-right evaluation of the three rng() calls. */
static int64_t gen_date(mt64 *s) {
  uint64_t y = 1992 + mt_next(s) % 7;
  uint64_t m = 1 + mt_next(s) % 12;
  uint64_t d = 1 + mt_next(s) % 28;
  return (int64_t)(y * 10000 + m * 100 + d);
}

/* ---------------- tables (column-major, whole table in RAM: oracle sizes only) ---------------- */
typedef struct {
  int ncols;
  const char *names[4];
  uint64_t rows;
  int64_t *cols[4];
} table_t;

static void table_alloc(table_t *t, uint64_t rows) {
  t->rows = rows;
  for (int c = 0; c < t->ncols; ++c) {
    t->cols[c] = (int64_t *)malloc((rows ? rows : 1) * 8);
  }
}
static void table_free(table_t *t) {
  for (int c = 0; c < t->ncols; ++c) free(t->cols[c]);
}

static void gen_customer(table_t *t, double scale, uint64_t seed) {
  const uint64_t rows = (uint64_t)(150000 * scale);
  mt64 s;
  mt_seed(&s, seed * 0x9E3779B97F4A7C15ULL + 11);
  t->ncols = 2;
  t->names[0] = "c_custkey";
  t->names[1] = "c_mktsegment";
  table_alloc(t, rows);
  for (uint64_t i = 0; i < rows; ++i) {
    t->cols[0][i] = (int64_t)i;
    t->cols[1][i] = (int64_t)(mt_next(&s) % 5);
  }
}

static void gen_orders(table_t *t, double scale, uint64_t seed) {
  const uint64_t customers = (uint64_t)(150000 * scale);
  const uint64_t rows = (uint64_t)(1500000 * scale);
  mt64 s;
  mt_seed(&s, seed * 0x9E3779B97F4A7C15ULL + 12);
  t->ncols = 4;
  t->names[0] = "o_orderkey";
  t->names[1] = "o_custkey";
  t->names[2] = "o_orderdate";
  t->names[3] = "o_shippriority";
  table_alloc(t, rows);
  for (uint64_t i = 0; i < rows; ++i) {
    t->cols[0][i] = (int64_t)i;
    t->cols[1][i] = customers > 0 ? (int64_t)(mt_next(&s) % customers) : 0;
    t->cols[2][i] = gen_date(&s);
    t->cols[3][i] = (int64_t)(mt_next(&s) % 5);
  }
}

static void gen_lineitem(table_t *t, double scale, uint64_t seed) {
  const uint64_t orders = (uint64_t)(1500000 * scale);
  const uint64_t rows = (uint64_t)(6000000 * scale);
  mt64 s;
  mt_seed(&s, seed * 0x9E3779B97F4A7C15ULL + 13);
  t->ncols = 4;
  t->names[0] = "l_orderkey";
  t->names[1] = "l_extendedprice";
  t->names[2] = "l_discount";
  t->names[3] = "l_shipdate";
  table_alloc(t, rows);
  for (uint64_t i = 0; i < rows; ++i) {
    t->cols[0][i] = orders > 0 ? (int64_t)(mt_next(&s) % orders) : 0;
    t->cols[1][i] = 90000 + (int64_t)(mt_next(&s) % 100000);
    t->cols[2][i] = (int64_t)(mt_next(&s) % 11);
    t->cols[3][i] = gen_date(&s);
  }
}

/* ---------------- PSTO writer ---------------- */
typedef struct { uint8_t *p; size_t n, cap; } buf_t;
static void bput(buf_t *b, const void *src, size_t n) {
  if (b->n + n > b->cap) {
    b->cap = (b->n + n) * 2 + 64;
    b->p = (uint8_t *)realloc(b->p, b->cap);
  }
  memcpy(b->p + b->n, src, n);
  b->n += n;
}
static void bu8(buf_t *b, uint8_t v) { bput(b, &v, 1); }
static void bu32(buf_t *b, uint32_t v) { bput(b, &v, 4); }
static void bu64(buf_t *b, uint64_t v) { bput(b, &v, 8); }

/* Writes rows [r ≡ node mod nodes] of t (nodes=1,node=0: all rows). Returns 0 on success. */
static int write_psto(const table_t *t, int node, int nodes, const char *path, uint64_t rg_bytes,
                      int codec) {
  FILE *f = fopen(path, "wb");
  if (!f) return -1;
  fwrite("PSTO", 1, 4, f);
  uint64_t offset = 4;
  const uint64_t total = t->rows > (uint64_t)node ? (t->rows - (uint64_t)node + (uint64_t)nodes - 1) / (uint64_t)nodes : 0;
  uint64_t rg_rows = rg_bytes / ((uint64_t)t->ncols * 8);
  if (rg_rows < 1) rg_rows = 1;
  buf_t footer = {0};
  bu32(&footer, 1);
  bu8(&footer, (uint8_t)codec);
  bu32(&footer, (uint32_t)t->ncols);
  for (int c = 0; c < t->ncols; ++c) {
    uint32_t len = (uint32_t)strlen(t->names[c]);
    bu32(&footer, len);
    bput(&footer, t->names[c], len);
    bu8(&footer, 0); /* Int64 */
  }
  const uint32_t ngroups = (uint32_t)((total + rg_rows - 1) / rg_rows);
  bu32(&footer, ngroups);
  int64_t *tmp = (int64_t *)malloc(rg_rows * 8);
  uLongf zcap = compressBound((uLong)(rg_rows * 8));
  uint8_t *z = (uint8_t *)malloc(zcap);
  for (uint32_t g = 0; g < ngroups; ++g) {
    const uint64_t lo = (uint64_t)g * rg_rows;
    const uint64_t n = (total - lo) < rg_rows ? (total - lo) : rg_rows;
    bu64(&footer, n);
    for (int c = 0; c < t->ncols; ++c) {
      int64_t mn = 0, mx = 0;
      for (uint64_t i = 0; i < n; ++i) {
        int64_t v = t->cols[c][(lo + i) * (uint64_t)nodes + (uint64_t)node];
        tmp[i] = v;
        if (i == 0 || v < mn) mn = v;
        if (i == 0 || v > mx) mx = v;
      }
      uint64_t csize = n * 8;
      const void *data = tmp;
      if (codec == 1) {
        uLongf zl = zcap;
        if (compress2(z, &zl, (const Bytef *)tmp, (uLong)(n * 8), 1) != Z_OK) return -2;
        csize = zl;
        data = z;
      }
      fwrite(data, 1, csize, f);
      bu64(&footer, offset);
      bu64(&footer, csize);
      bu64(&footer, n * 8);
      bu64(&footer, (uint64_t)mn);
      bu64(&footer, (uint64_t)mx);
      offset += csize;
    }
  }
  fwrite(footer.p, 1, footer.n, f);
  uint64_t flen = footer.n;
  fwrite(&flen, 8, 1, f);
  fwrite("PSTO", 1, 4, f);
  free(footer.p);
  free(tmp);
  free(z);
  return fclose(f) == 0 ? 0 : -3;
}

static void mkdir_p(const char *dir) {
  char tmp[4096];
  snprintf(tmp, sizeof tmp, "%s", dir);
  for (char *p = tmp + 1; *p; ++p)
    if (*p == '/') {
      *p = 0;
      mkdir(tmp, 0755);
      *p = '/';
    }
  mkdir(tmp, 0755);
}

/* gen_workload(kind=tpch) restated: bench.cpp:85-114. Returns 0 on success. */
int orc_gen_tpch(const char *out_dir, double scale, int nodes, int devices, uint64_t seed,
                 int codec, uint64_t rg_bytes) {
  if (nodes < 1 || devices < 1) return -1;
  char dir[4096], path[4600];
  table_t t;
  memset(&t, 0, sizeof t);
  gen_customer(&t, scale, seed);
  snprintf(dir, sizeof dir, "%s/dev%d", out_dir, 0 % devices);
  mkdir_p(dir);
  snprintf(path, sizeof path, "%s/customer.psto", dir);
  if (write_psto(&t, 0, 1, path, rg_bytes, codec)) return -2;
  table_free(&t);
  const char *names[2] = {"orders", "lineitem"};
  for (int k = 0; k < 2; ++k) {
    memset(&t, 0, sizeof t);
    if (k == 0) gen_orders(&t, scale, seed); else gen_lineitem(&t, scale, seed);
    for (int node = 0; node < nodes; ++node) {
      snprintf(dir, sizeof dir, "%s/dev%d", out_dir, (k + node) % devices);
      mkdir_p(dir);
      snprintf(path, sizeof path, "%s/%s.node%d.psto", dir, names[k], node);
      if (write_psto(&t, node, nodes, path, rg_bytes, codec)) return -3;
    }
    table_free(&t);
  }
  return 0;
}
