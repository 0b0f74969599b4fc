/*
 * irismpc oracle — CPU restatement of the reference hot path (TEST
 * INFRASTRUCTURE ONLY; see irismpc_oracle.h for who may use it).
 *
 * Every function cites the reference file:line (under /root/reference/proj)
 * whose behaviour it restates.  Parties are simulated in component form.
 */
#include "irismpc_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ====================================================================== */
/* ChaCha12 counter PRF — prf.hpp:35-69                                    */
/* ====================================================================== */

static inline uint32_t rotl32(uint32_t x, int n) { return (x << n) | (x >> (32 - n)); }

#define QR(a, b, c, d)                 \
  do {                                 \
    a += b; d ^= a; d = rotl32(d, 16); \
    c += d; b ^= c; b = rotl32(b, 12); \
    a += b; d ^= a; d = rotl32(d, 8);  \
    c += d; b ^= c; b = rotl32(b, 7);  \
  } while (0)

/* detail::chacha_block (prf.hpp:46-69): 128-bit key duplicated into words
 * 4-11, 64-bit block counter in 12-13, 64-bit stream id in 14-15, 6 double
 * rounds, feed-forward. */
void orc_chacha_block(const uint8_t seed[16], uint64_t block, uint64_t stream,
                      uint32_t out[16]) {
  uint32_t key[4];
  memcpy(key, seed, 16);
  uint32_t st[16] = {0x61707865u, 0x3320646eu, 0x79622d32u, 0x6b206574u,
                     key[0], key[1], key[2], key[3],
                     key[0], key[1], key[2], key[3],
                     (uint32_t)block, (uint32_t)(block >> 32),
                     (uint32_t)stream, (uint32_t)(stream >> 32)};
  uint32_t x[16];
  memcpy(x, st, sizeof(st));
  for (int r = 0; r < 6; ++r) {
    QR(x[0], x[4], x[8], x[12]);
    QR(x[1], x[5], x[9], x[13]);
    QR(x[2], x[6], x[10], x[14]);
    QR(x[3], x[7], x[11], x[15]);
    QR(x[0], x[5], x[10], x[15]);
    QR(x[1], x[6], x[11], x[12]);
    QR(x[2], x[7], x[8], x[13]);
    QR(x[3], x[4], x[9], x[14]);
  }
  for (int i = 0; i < 16; ++i) out[i] = x[i] + st[i];
}

/* CtrPrf::derive (prf.hpp:106-112) */
void orc_derive(const uint8_t parent[16], uint64_t tag, uint8_t out[16]) {
  uint32_t blk[16];
  orc_chacha_block(parent, tag, 0xD5A1u, blk);
  memcpy(out, blk, 16);
}

/* CtrPrf::seed_from_u64 (prf.hpp:114-118) */
void orc_seed_from_u64(uint64_t v, uint8_t out[16]) {
  uint8_t s[16] = {0};
  memcpy(s, &v, 8);
  orc_derive(s, 0, out);
}

/* CtrPrf stream element: refill() memcpy's the 16 u32 words into 8 u64
 * (prf.hpp:123-128), so element idx is word idx%8 of block idx/8. */
uint64_t orc_stream_at(const uint8_t seed[16], uint64_t stream, uint64_t idx) {
  uint32_t blk[16];
  orc_chacha_block(seed, idx / 8, stream, blk);
  const unsigned w = (unsigned)(idx % 8);
  return (uint64_t)blk[2 * w] | ((uint64_t)blk[2 * w + 1] << 32);
}

/* Random-access reader with a one-block cache (test-speed helper only). */
typedef struct {
  const uint8_t* seed;
  uint64_t cached;
  int valid;
  uint64_t buf[8];
} prf_reader;

static void reader_init(prf_reader* r, const uint8_t* seed) {
  r->seed = seed;
  r->valid = 0;
}

static uint64_t reader_at(prf_reader* r, uint64_t idx) {
  const uint64_t blk = idx / 8;
  if (!r->valid || r->cached != blk) {
    uint32_t out[16];
    orc_chacha_block(r->seed, blk, 0, out);
    memcpy(r->buf, out, 64);
    r->cached = blk;
    r->valid = 1;
  }
  return r->buf[idx % 8];
}

/* ====================================================================== */
/* Rng — prf.hpp:138-167                                                   */
/* ====================================================================== */

struct orc_rng {
  uint8_t seed[16];
  uint64_t pos; /* next element index of stream 0 */
  prf_reader rd;
};

orc_rng* orc_rng_new_seed(const uint8_t seed[16]) {
  orc_rng* r = (orc_rng*)calloc(1, sizeof(orc_rng));
  memcpy(r->seed, seed, 16);
  reader_init(&r->rd, r->seed);
  return r;
}

orc_rng* orc_rng_new(uint64_t seed) {
  uint8_t s[16];
  orc_seed_from_u64(seed, s);
  return orc_rng_new_seed(s);
}

/* sub_rng (cluster.cpp:24-26) */
orc_rng* orc_rng_sub(uint64_t seed, uint64_t tag) {
  uint8_t s[16], d[16];
  orc_seed_from_u64(seed, s);
  orc_derive(s, tag, d);
  return orc_rng_new_seed(d);
}

void orc_rng_free(orc_rng* r) { free(r); }

uint64_t orc_rng_next(orc_rng* r) { return reader_at(&r->rd, r->pos++); }

uint64_t orc_rng_position(const orc_rng* r) { return r->pos; }

/* Rng::below (prf.hpp:145-152): rejection below the largest multiple. */
uint64_t orc_rng_below(orc_rng* r, uint64_t bound) {
  const uint64_t lim = ~(uint64_t)0 - (~(uint64_t)0) % bound;
  uint64_t v;
  do {
    v = orc_rng_next(r);
  } while (v >= lim);
  return v % bound;
}

/* Rng::with_probability (prf.hpp:155-157) */
int orc_rng_with_probability(orc_rng* r, double p) {
  return (double)(orc_rng_next(r) >> 11) * 0x1.0p-53 < p;
}

/* BitVec::random (iris.hpp:69-73) */
static void bitvec_random(orc_rng* r, uint32_t l, double density, uint64_t* w) {
  const uint32_t nw = (l + 63) / 64;
  memset(w, 0, nw * sizeof(uint64_t));
  for (uint32_t i = 0; i < l; ++i) {
    if (orc_rng_with_probability(r, density)) w[i / 64] |= (uint64_t)1 << (i % 64);
  }
}

/* random_record (iris.hpp:294-296): IrisRecord(BitVec::random(l, rng),
 * BitVec::random(l, rng, d)); GCC evaluates the mask argument first. */
void orc_rng_record(orc_rng* r, uint32_t l, double mask_density, uint64_t* code,
                    uint64_t* mask) {
  bitvec_random(r, l, mask_density, mask);
  bitvec_random(r, l, 0.5, code);
}

/* deal_seeds (rep3.hpp:116-122) over Rng(derive(seed_from_u64(seed), 0x5eed))
 * (cluster.hpp:35-36). */
void orc_party_seeds(uint64_t master, uint8_t out[48]) {
  uint8_t s[16], d[16];
  orc_seed_from_u64(master, s);
  orc_derive(s, 0x5eed, d);
  orc_rng* r = orc_rng_new_seed(d);
  for (int i = 0; i < 48; ++i) out[i] = (uint8_t)orc_rng_next(r);
  orc_rng_free(r);
}

/* ====================================================================== */
/* Galois ring Z_2^K[X]/(X^2-X-1), K = 16 or 32 — galois.hpp:30-128         */
/* ====================================================================== */

typedef struct { uint32_t c0, c1; } gr;

static inline uint32_t kmask(unsigned K) { return K == 32 ? 0xFFFFFFFFu : ((1u << K) - 1); }

static gr gr_mul(gr a, gr b, unsigned K) {
  const uint32_t m = kmask(K);
  gr r;
  r.c0 = (uint32_t)((uint64_t)a.c0 * b.c0 + (uint64_t)a.c1 * b.c1) & m;
  r.c1 = (uint32_t)((uint64_t)a.c0 * b.c1 + (uint64_t)a.c1 * b.c0 + (uint64_t)a.c1 * b.c1) & m;
  return r;
}
static gr gr_sub(gr a, gr b, unsigned K) {
  gr r = {(a.c0 - b.c0) & kmask(K), (a.c1 - b.c1) & kmask(K)};
  return r;
}
static gr gr_add(gr a, gr b, unsigned K) {
  gr r = {(a.c0 + b.c0) & kmask(K), (a.c1 + b.c1) & kmask(K)};
  return r;
}

/* gr_inverse (galois.hpp:66-87): F_4 seed then Newton y <- y(2 - a y). */
static gr gr_inverse(gr a, unsigned K) {
  const unsigned p0 = a.c0 & 1, p1 = a.c1 & 1;
  gr y;
  if (p1 == 0) {
    y.c0 = 1; y.c1 = 0;
  } else if (p0 == 0) {
    y.c0 = 1; y.c1 = 1;
  } else {
    y.c0 = 0; y.c1 = 1;
  }
  const gr two = {2, 0};
  for (unsigned correct = 1; correct < K; correct *= 2) y = gr_mul(y, gr_sub(two, gr_mul(a, y, K), K), K);
  return y;
}

/* party_lagrange_at_zero over the exceptional points {1, X, 1+X}
 * (galois.hpp:92-128). */
void orc_lambda(unsigned K, uint32_t out[6]) {
  const gr xs[3] = {{1, 0}, {0, 1}, {1, 1}};
  for (int i = 0; i < 3; ++i) {
    gr num = {1, 0}, den = {1, 0};
    for (int j = 0; j < 3; ++j) {
      if (j == i) continue;
      num = gr_mul(num, xs[j], K);
      den = gr_mul(den, gr_sub(xs[j], xs[i], K), K);
    }
    const gr li = gr_mul(num, gr_inverse(den, K), K);
    out[2 * i] = li.c0;
    out[2 * i + 1] = li.c1;
  }
}

void orc_lambda16(uint16_t out[6]) {
  uint32_t l32[6];
  orc_lambda(16, l32);
  for (int i = 0; i < 6; ++i) out[i] = (uint16_t)l32[i];
}

/* ====================================================================== */
/* Variant widths (shares.hpp:28-48) and dealer (shares.hpp:52-130,        */
/* shares.cpp:49-90)                                                       */
/* ====================================================================== */

unsigned orc_code_bits(int variant) { return variant == ORC_NO_LIFT ? 32 : 16; }
unsigned orc_mask_bits(int variant) {
  switch (variant) {
    case ORC_PLAIN_MASK: return 0;
    case ORC_MPC_LIFT: return 16;
    default: return 32;
  }
}
unsigned orc_cmp_bits(int variant) { return variant == ORC_PLAIN_MASK ? 16 : 32; }

/* code_record_bytes / mask_record_bytes (shares.cpp:49-59) */
size_t orc_code_record_bytes(int backend, int variant, uint32_t l) {
  const size_t w = orc_code_bits(variant) / 8;
  return backend == ORC_REPLICATED ? (size_t)l * 2 * w : (size_t)(l / 2) * 2 * w;
}
size_t orc_mask_record_bytes(int backend, int variant, uint32_t l) {
  const unsigned km = orc_mask_bits(variant);
  if (km == 0) return l / 8;
  const size_t w = km / 8;
  return backend == ORC_REPLICATED ? (size_t)l * 2 * w : (size_t)(l / 2) * 2 * w;
}

static inline void putw(uint8_t** p, uint32_t v, unsigned K) {
  for (unsigned b = 0; b < K / 8; ++b) (*p)[b] = (uint8_t)(v >> (8 * b));
  *p += K / 8;
}
static inline uint32_t getw(const uint8_t* p, unsigned K) {
  uint32_t v = 0;
  for (unsigned b = 0; b < K / 8; ++b) v |= (uint32_t)p[b] << (8 * b);
  return v;
}

static inline int bit_at(const uint64_t* w, uint32_t i) { return (int)((w[i / 64] >> (i % 64)) & 1); }

/* emit_rep_record (shares.hpp:63-73) with share<K> (rep3.hpp:74-80) */
static void emit_rep(const uint32_t* vals, uint32_t n, unsigned K, orc_rng* rng, uint8_t** o) {
  const uint32_t m = kmask(K);
  for (uint32_t i = 0; i < n; ++i) {
    const uint32_t x1 = (uint32_t)orc_rng_next(rng) & m;
    const uint32_t x2 = (uint32_t)orc_rng_next(rng) & m;
    const uint32_t x3 = (vals[i] - x1 - x2) & m;
    putw(&o[0], x1, K); putw(&o[0], x3, K);
    putw(&o[1], x2, K); putw(&o[1], x1, K);
    putw(&o[2], x3, K); putw(&o[2], x2, K);
  }
}

/* emit_gr_record (shares.hpp:75-85) with shamir_share_packed (shamir.hpp:46-59).
 * `Gr<K> r(rng.ring(), rng.ring())` gives the FIRST draw to c1 under GCC
 * (SURVEY.md A.4).  Share at point x_p: g + r * x_p with x = {1, X, 1+X}. */
static void emit_gr(const uint32_t* vals, uint32_t n, unsigned K, orc_rng* rng, uint8_t** o) {
  const gr pts[3] = {{1, 0}, {0, 1}, {1, 1}};
  const uint32_t m = kmask(K);
  for (uint32_t i = 0; i < n / 2; ++i) {
    gr g = {vals[2 * i], vals[2 * i + 1]};
    gr r;
    r.c1 = (uint32_t)orc_rng_next(rng) & m;
    r.c0 = (uint32_t)orc_rng_next(rng) & m;
    for (int p = 0; p < 3; ++p) {
      const gr sh = gr_add(g, gr_mul(r, pts[p], K), K);
      putw(&o[p], sh.c0, K);
      putw(&o[p], sh.c1, K);
    }
  }
}

/* emit_record (shares.cpp:61-74): masked code entries m - 2(c&m) (iris.hpp:108-112)
 * at code_bits, then the mask: shares at mask_bits, or l/8 plain mask bytes
 * identical for all parties (emit_mask_bits, shares.hpp:87-95). */
void orc_deal_payload_v(int backend, int variant, uint32_t l, uint64_t nrec, const uint64_t* codes,
                        const uint64_t* masks, orc_rng* rng, uint8_t* out1, uint8_t* out2, uint8_t* out3) {
  const uint32_t wl = (l + 63) / 64;
  const unsigned KH = orc_code_bits(variant), KM = orc_mask_bits(variant);
  uint32_t* cv = (uint32_t*)malloc(sizeof(uint32_t) * l);
  uint32_t* mv = (uint32_t*)malloc(sizeof(uint32_t) * l);
  uint8_t* o[3] = {out1, out2, out3};
  for (uint64_t r = 0; r < nrec; ++r) {
    const uint64_t* c = codes + r * wl;
    const uint64_t* m = masks + r * wl;
    for (uint32_t i = 0; i < l; ++i) {
      const int mb = bit_at(m, i), cb = bit_at(c, i) & mb;
      cv[i] = (uint32_t)(mb - 2 * cb) & kmask(KH);
      mv[i] = (uint32_t)mb;
    }
    if (backend == ORC_REPLICATED)
      emit_rep(cv, l, KH, rng, o);
    else
      emit_gr(cv, l, KH, rng, o);
    if (KM == 0) {
      for (int p = 0; p < 3; ++p)
        for (uint32_t i = 0; i < l / 8; ++i) o[p][i] = (uint8_t)(m[i / 8] >> (8 * (i % 8)));
      for (int p = 0; p < 3; ++p) o[p] += l / 8;
    } else if (backend == ORC_REPLICATED) {
      emit_rep(mv, l, KM, rng, o);
    } else {
      emit_gr(mv, l, KM, rng, o);
    }
  }
  free(cv);
  free(mv);
}

/* legacy entry: mpc-lift widths */
size_t orc_code_record_bytes16(int backend, uint32_t l) { return orc_code_record_bytes(backend, ORC_MPC_LIFT, l); }
void orc_deal_payload(int backend, uint32_t l, uint64_t nrec, const uint64_t* codes, const uint64_t* masks,
                      orc_rng* rng, uint8_t* out1, uint8_t* out2, uint8_t* out3) {
  orc_deal_payload_v(backend, ORC_MPC_LIFT, l, nrec, codes, masks, rng, out1, out2, out3);
}

/* ====================================================================== */
/* Engine — engine.cpp / engine.hpp / circuits.hpp / convert.hpp           */
/* ====================================================================== */

uint32_t orc_match_a(double ratio) {
  /* MatchParams::make (iris.hpp:163-174) with m = 16 */
  const uint32_t b = 1u << 16;
  long long a = llround((1.0 - 2.0 * ratio) * (double)b);
  if (a > (long long)b) a = b;
  return (uint32_t)a;
}

/* EngineConfig::validate (engine.cpp:21-34) */
int orc_validate(const orc_config* cfg) {
  if (cfg->l == 0 || cfg->l % 8 != 0) return 4;
  if (cfg->a > cfg->b) return 4;
  if (cfg->variant == ORC_PLAIN_MASK) {
    /* check_public_mask_bound(l, 16) (iris.hpp:190-196) */
    const uint64_t t = (uint64_t)1 << 16;
    if (!(cfg->l < t / 4 && cfg->l < t - (t >> 1))) return 4;
  } else {
    if (cfg->b != (1u << 16)) return 4;
    /* check_shared_mask_bound(l, b, 32) (iris.hpp:199-205) */
    const uint64_t t = (uint64_t)1 << 32;
    const uint64_t bl = (uint64_t)cfg->b * cfg->l;
    if (!(bl < t / 4 && bl < t - (t >> 1))) return 4;
  }
  if (cfg->rotations % 2 == 0) return 4;
  if (cfg->backend == ORC_SHAMIR && cfg->rotations > 1 && (cfg->l / 64) % 2 != 0) return 4;
  return 0;
}

uint64_t orc_lane_count(uint32_t persons, uint64_t s, uint32_t rotations, int membership) {
  if (membership) return s;
  const uint64_t blocks = 2ull * persons * rotations;
  const uint64_t pairs = (uint64_t)persons * (persons ? persons - 1 : 0) / 2 * 4 * rotations;
  return blocks * s + pairs;
}

/* Per-party parsed instance (engine.hpp:141-197) at width K.  rep: sum/prev;
 * shamir: a = lambda-scaled [lc0 | lc1], b = raw [c0 | c1]. */
typedef struct {
  uint32_t* a;
  uint32_t* b;
} inst;

/* parse_rep_inst (engine.hpp:162-176) / parse_gr_inst (engine.hpp:178-197) */
static void parse_inst(int backend, const uint8_t* p, uint32_t l, unsigned K, const gr lambda, inst* out) {
  const unsigned w = K / 8;
  const uint32_t m = kmask(K);
  out->a = (uint32_t*)malloc(sizeof(uint32_t) * l);
  out->b = (uint32_t*)malloc(sizeof(uint32_t) * l);
  if (backend == ORC_REPLICATED) {
    for (uint32_t i = 0; i < l; ++i) {
      const uint32_t own = getw(p + 2 * w * i, K);
      const uint32_t prev = getw(p + 2 * w * i + w, K);
      out->a[i] = (own + prev) & m;
      out->b[i] = prev;
    }
  } else {
    const uint32_t h = l / 2;
    for (uint32_t i = 0; i < h; ++i) {
      gr g = {getw(p + 2 * w * i, K), getw(p + 2 * w * i + w, K)};
      const gr lg = gr_mul(lambda, g, K);
      out->a[i] = lg.c0;
      out->a[h + i] = lg.c1;
      out->b[i] = g.c0;
      out->b[h + i] = g.c1;
    }
  }
}

static void free_inst(inst* x) {
  free(x->a);
  free(x->b);
}

/* rotate_vec (engine.hpp:126-136): out[(i + by) mod n] = v[i]. */
static void rotate(const uint32_t* v, uint32_t n, int64_t by, uint32_t* out) {
  int64_t s = n ? by % (int64_t)n : 0;
  if (s < 0) s += n;
  for (uint32_t i = 0; i < n; ++i) out[(i + (uint64_t)s) % n] = v[i];
}

/* RepInst::rotated / GrInst::rotated (engine.hpp:149-159) */
static void rotate_inst(int backend, const inst* x, uint32_t l, int64_t by, inst* out) {
  out->a = (uint32_t*)malloc(sizeof(uint32_t) * l);
  out->b = (uint32_t*)malloc(sizeof(uint32_t) * l);
  if (backend == ORC_REPLICATED) {
    rotate(x->a, l, by, out->a);
    rotate(x->b, l, by, out->b);
  } else {
    const uint32_t h = l / 2;
    const int64_t bp = by / 2;
    rotate(x->a, h, bp, out->a);
    rotate(x->a + h, h, bp, out->a + h);
    rotate(x->b, h, bp, out->b);
    rotate(x->b + h, h, bp, out->b + h);
  }
}

/* dot_prep_row (kernels.hpp:38-48) / dot_gr_ct_row (kernels.hpp:52-62), mod 2^K */
static uint32_t dot_row(int backend, const uint32_t* xa, const uint32_t* xb, const inst* y, uint32_t l, unsigned K) {
  uint64_t acc = 0;
  if (backend == ORC_REPLICATED) {
    for (uint32_t i = 0; i < l; ++i) {
      acc += (uint64_t)xa[i] * y->a[i];
      acc -= (uint64_t)xb[i] * y->b[i];
    }
  } else {
    for (uint32_t i = 0; i < l; ++i) acc += (uint64_t)xa[i] * y->b[i];
  }
  return (uint32_t)acc & kmask(K);
}

/* parse_mask_bits (engine.hpp:199-206) + BitVec::rotated (iris.hpp:56-66) */
static void mask_bits(const uint8_t* p, uint32_t l, uint64_t* w) {
  const uint32_t wl = (l + 63) / 64;
  memset(w, 0, sizeof(uint64_t) * wl);
  for (uint32_t i = 0; i < l / 8; ++i) w[i / 8] |= (uint64_t)p[i] << (8 * (i % 8));
}
static void rotate_bits(const uint64_t* in, uint32_t l, int64_t by, uint64_t* out) {
  const uint32_t wl = (l + 63) / 64;
  memset(out, 0, sizeof(uint64_t) * wl);
  int64_t s = l ? by % (int64_t)l : 0;
  if (s < 0) s += l;
  for (uint32_t i = 0; i < l; ++i)
    if ((in[i / 64] >> (i % 64)) & 1) {
      const uint32_t j = (uint32_t)((i + (uint64_t)s) % l);
      out[j / 64] |= (uint64_t)1 << (j % 64);
    }
}
static int64_t popcount_and(const uint64_t* a, const uint64_t* b, uint32_t l) {
  int64_t c = 0;
  for (uint32_t i = 0; i < (l + 63) / 64; ++i) c += __builtin_popcountll(a[i] & b[i]);
  return c;
}

/* ---- bit-sliced 3-party simulation (circuits.hpp) ---------------------- */

static uint64_t ceil_div(uint64_t a, uint64_t b) { return (a + b - 1) / b; }

typedef struct {
  uint64_t* c[3]; /* XOR components, W words each */
} brow;

static brow brow_new(uint64_t W) {
  brow r;
  for (int p = 0; p < 3; ++p) r.c[p] = (uint64_t*)calloc(W ? W : 1, sizeof(uint64_t));
  return r;
}
static void brow_free(brow* r) {
  for (int p = 0; p < 3; ++p) free(r->c[p]);
}
static void brow_xor(brow* dst, const brow* a, const brow* b, uint64_t W) {
  for (int p = 0; p < 3; ++p)
    for (uint64_t w = 0; w < W; ++w) dst->c[p][w] = a->c[p][w] ^ b->c[p][w];
}
static void brow_copy(brow* dst, const brow* a, uint64_t W) {
  for (int p = 0; p < 3; ++p) memcpy(dst->c[p], a->c[p], W * sizeof(uint64_t));
}

typedef struct {
  const uint8_t* seed[3];
  prf_reader rd[3];
  uint64_t pos[3];
} prf_state;

/* and_layer gate (circuits.hpp:92-131) in component form:
 * z_p = x_p y_p ^ x_{p-1} y_p ^ x_p y_{p-1} ^ F(seed_p) ^ F(seed_{p-1}),
 * one zero_word per 64-lane word at stream index base + w, dead lanes masked
 * (circuits.hpp:82-87). */
static void and_gate(prf_state* ps, const brow* x, const brow* y, brow* z, uint64_t words,
                     uint64_t lanes, const uint64_t base[3]) {
  for (uint64_t w = 0; w < words; ++w) {
    uint64_t f[3];
    for (int k = 0; k < 3; ++k) f[k] = reader_at(&ps->rd[k], base[k] + w);
    uint64_t zc[3];
    for (int p = 0; p < 3; ++p) {
      const int q = (p + 2) % 3; /* prev party's component */
      zc[p] = (x->c[p][w] & y->c[p][w]) ^ (x->c[q][w] & y->c[p][w]) ^
              (x->c[p][w] & y->c[q][w]) ^ f[p] ^ f[q];
    }
    for (int p = 0; p < 3; ++p) z->c[p][w] = zc[p];
  }
  if (words && lanes % 64) {
    const uint64_t m = ((uint64_t)1 << (lanes % 64)) - 1;
    for (int p = 0; p < 3; ++p) z->c[p][words - 1] &= m;
  }
}

/* or_tree_batch (circuits.hpp:387-434): every group folds level by level
 * (lo = first ceil(N/2) lanes, hi = the rest, lo ^ hi ^ AND(lo, hi) over nb
 * lanes), all groups of a level in one and_layer round whose gates draw
 * ceil(nb/64) words each in group order.  grp[g] / gl[g] are replaced by the
 * one-lane results. */
static void or_tree_groups(prf_state* ps, brow* grp, uint64_t* gl, uint32_t ngroups, uint64_t* rounds,
                           uint64_t* bytes) {
  for (;;) {
    int progress = 0;
    uint64_t used = 0;
    for (uint32_t g = 0; g < ngroups; ++g) {
      if (gl[g] <= 1) continue;
      progress = 1;
      const uint64_t na = (gl[g] + 1) / 2, nb = gl[g] - na;
      const uint64_t wa = ceil_div(na, 64), wb = ceil_div(nb, 64);
      brow lo = brow_new(wa), hi = brow_new(wa), t = brow_new(wa);
      for (uint64_t i = 0; i < na; ++i)
        for (int p = 0; p < 3; ++p)
          if ((grp[g].c[p][i / 64] >> (i % 64)) & 1) lo.c[p][i / 64] |= (uint64_t)1 << (i % 64);
      for (uint64_t i = 0; i < nb; ++i)
        for (int p = 0; p < 3; ++p) {
          const uint64_t src = na + i;
          if ((grp[g].c[p][src / 64] >> (src % 64)) & 1) hi.c[p][i / 64] |= (uint64_t)1 << (i % 64);
        }
      uint64_t base[3];
      for (int q = 0; q < 3; ++q) base[q] = ps->pos[q] + used;
      and_gate(ps, &lo, &hi, &t, wb, nb, base);
      used += wb;
      *bytes += ceil_div(nb, 8);
      for (int p = 0; p < 3; ++p)
        for (uint64_t w = 0; w < wa; ++w) lo.c[p][w] ^= hi.c[p][w] ^ (w < wb ? t.c[p][w] : 0);
      brow_free(&grp[g]);
      grp[g] = lo;
      gl[g] = na;
      brow_free(&hi);
      brow_free(&t);
    }
    if (!progress) break;
    for (int q = 0; q < 3; ++q) ps->pos[q] += used;
    ++*rounds;
  }
}

int orc_or_tree_batch(const uint8_t seeds[48], const uint64_t* stream_start, uint32_t ngroups,
                      const uint64_t* lens, const uint8_t* comps, uint64_t total, uint8_t* agg,
                      uint64_t* stream_pos) {
  prf_state ps;
  for (int k = 0; k < 3; ++k) {
    ps.seed[k] = seeds + 16 * k;
    reader_init(&ps.rd[k], ps.seed[k]);
    ps.pos[k] = stream_start ? stream_start[k] : 0;
  }
  brow* grp = (brow*)malloc(sizeof(brow) * (ngroups ? ngroups : 1));
  uint64_t* gl = (uint64_t*)malloc(sizeof(uint64_t) * (ngroups ? ngroups : 1));
  uint64_t off = 0;
  for (uint32_t g = 0; g < ngroups; ++g) {
    gl[g] = lens[g];
    grp[g] = brow_new(ceil_div(lens[g], 64));
    for (uint64_t i = 0; i < lens[g]; ++i)
      for (int p = 0; p < 3; ++p)
        if (comps[p * total + off + i] & 1) grp[g].c[p][i / 64] |= (uint64_t)1 << (i % 64);
    off += lens[g];
  }
  uint64_t rounds = 0, bytes = 0;
  or_tree_groups(&ps, grp, gl, ngroups, &rounds, &bytes);
  for (uint32_t g = 0; g < ngroups; ++g) {
    for (int p = 0; p < 3; ++p) agg[p * ngroups + g] = gl[g] == 0 ? 0 : (uint8_t)(grp[g].c[p][0] & 1);
    brow_free(&grp[g]);
  }
  if (stream_pos)
    for (int k = 0; k < 3; ++k) stream_pos[k] = ps.pos[k];
  free(grp);
  free(gl);
  return 0;
}

/* bit_extract_sum (circuits.hpp:202-296) for summand bit matrices rows[k][j]
 * of component k (share_split, circuits.hpp:152-172: summand k is binary
 * shared with only component k non-zero).  indices ascending as given. */
static void bit_extract(prf_state* ps, uint64_t n, uint64_t W, unsigned K, uint64_t* const* xs[3],
                        const unsigned* idx, unsigned nidx, brow* result) {
  typedef struct {
    unsigned m;
    brow* s;
    brow* carry;
    brow chain, u, v, res;
  } instance;
  instance inst[4];
  brow* a_rows[3];
  unsigned maxj = 0;
  for (unsigned k = 0; k < nidx; ++k) maxj = idx[k] > maxj ? idx[k] : maxj;
  for (int k = 0; k < 3; ++k) {
    a_rows[k] = (brow*)malloc(sizeof(brow) * (maxj + 1));
    for (unsigned j = 0; j <= maxj; ++j) {
      a_rows[k][j] = brow_new(W);
      if (j < K) memcpy(a_rows[k][j].c[k], xs[k][j], W * sizeof(uint64_t));
    }
  }
  for (unsigned k = 0; k < nidx; ++k) {
    instance* I = &inst[k];
    I->m = idx[k];
    I->s = (brow*)malloc(sizeof(brow) * (I->m + 1));
    I->carry = (brow*)malloc(sizeof(brow) * (I->m ? I->m : 1));
    for (unsigned j = 0; j <= I->m; ++j) {
      I->s[j] = brow_new(W);
      brow_xor(&I->s[j], &a_rows[0][j], &a_rows[1][j], W);
      brow_xor(&I->s[j], &I->s[j], &a_rows[2][j], W);
    }
    I->chain = brow_new(W);
    I->u = brow_new(W);
    I->v = brow_new(W);
    I->res = brow_new(W);
  }
  /* FA layer: one round, gates in instance order then j (circuits.hpp:243-259) */
  uint64_t g = 0;
  brow t1 = brow_new(W), t2 = brow_new(W);
  for (unsigned k = 0; k < nidx; ++k) {
    instance* I = &inst[k];
    for (unsigned j = 0; j < I->m; ++j) {
      brow_xor(&t1, &a_rows[0][j], &a_rows[2][j], W);
      brow_xor(&t2, &a_rows[1][j], &a_rows[2][j], W);
      I->carry[j] = brow_new(W);
      uint64_t base[3];
      for (int q = 0; q < 3; ++q) base[q] = ps->pos[q] + g * W;
      and_gate(ps, &t1, &t2, &I->carry[j], W, n, base);
      brow_xor(&I->carry[j], &I->carry[j], &a_rows[2][j], W);
      ++g;
    }
  }
  /* ripple chain (circuits.hpp:263-288) */
  for (unsigned t = 1; t + 1 <= maxj; ++t) {
    for (unsigned k = 0; k < nidx; ++k) {
      instance* I = &inst[k];
      if (t + 1 > I->m) continue;
      if (t == 1) {
        brow_copy(&I->u, &I->s[t], W);
        brow_copy(&I->v, &I->carry[t - 1], W);
      } else {
        brow_xor(&I->u, &I->s[t], &I->chain, W);
        brow_xor(&I->v, &I->carry[t - 1], &I->chain, W);
      }
      uint64_t base[3];
      for (int q = 0; q < 3; ++q) base[q] = ps->pos[q] + g * W;
      and_gate(ps, &I->u, &I->v, &I->res, W, n, base);
      ++g;
      if (t == 1)
        brow_copy(&I->chain, &I->res, W);
      else
        brow_xor(&I->chain, &I->res, &I->chain, W);
    }
  }
  for (unsigned k = 0; k < nidx; ++k) {
    instance* I = &inst[k];
    if (I->m == 0) {
      brow_copy(&result[k], &I->s[0], W);
    } else {
      brow_xor(&result[k], &I->s[I->m], &I->carry[I->m - 1], W);
      if (I->m >= 2) brow_xor(&result[k], &result[k], &I->chain, W);
    }
  }
  for (int q = 0; q < 3; ++q) ps->pos[q] += g * W;
  for (unsigned k = 0; k < nidx; ++k) {
    instance* I = &inst[k];
    for (unsigned j = 0; j <= I->m; ++j) brow_free(&I->s[j]);
    for (unsigned j = 0; j < I->m; ++j) brow_free(&I->carry[j]);
    free(I->s);
    free(I->carry);
    brow_free(&I->chain);
    brow_free(&I->u);
    brow_free(&I->v);
    brow_free(&I->res);
  }
  for (int k = 0; k < 3; ++k) {
    for (unsigned j = 0; j <= maxj; ++j) brow_free(&a_rows[k][j]);
    free(a_rows[k]);
  }
  brow_free(&t1);
  brow_free(&t2);
}

/* share_split (circuits.hpp:152-172): bit j of component k, 64 lanes/word */
static uint64_t*** share_split(const uint32_t* const comps[3], uint64_t n, uint64_t W, unsigned K) {
  uint64_t*** xs = (uint64_t***)malloc(sizeof(uint64_t**) * 3);
  for (int k = 0; k < 3; ++k) {
    xs[k] = (uint64_t**)malloc(sizeof(uint64_t*) * K);
    for (unsigned j = 0; j < K; ++j) xs[k][j] = (uint64_t*)calloc(W ? W : 1, sizeof(uint64_t));
    for (uint64_t i = 0; i < n; ++i) {
      const uint32_t v = comps[k][i];
      for (unsigned j = 0; j < K; ++j)
        if ((v >> j) & 1) xs[k][j][i / 64] |= (uint64_t)1 << (i % 64);
    }
  }
  return xs;
}
static void free_split(uint64_t*** xs, unsigned K) {
  for (int k = 0; k < 3; ++k) {
    for (unsigned j = 0; j < K; ++j) free(xs[k][j]);
    free(xs[k]);
  }
  free(xs);
}

/* bit_inject<W> (convert.hpp:84-155) in component form.  Per lane i:
 * c1 = F(seed_1, pos1+i), (c3, w0, w1) = F(seed_3, pos3+3i+{0,1,2});
 * P2 recovers c2 = m_{x2} = (x1^x2^x3) - c1 - c3 through the 3OT; the OT
 * pads w0/w1 are consumed but cancel out of every share. */
static void bit_inject(prf_state* ps, const brow* bits, uint64_t n, unsigned width, uint32_t* out[3]) {
  const uint32_t mask = (1u << width) - 1;
  for (uint64_t i = 0; i < n; ++i) {
    const unsigned x1 = (bits->c[0][i / 64] >> (i % 64)) & 1;
    const unsigned x2 = (bits->c[1][i / 64] >> (i % 64)) & 1;
    const unsigned x3 = (bits->c[2][i / 64] >> (i % 64)) & 1;
    const uint32_t c1 = (uint32_t)reader_at(&ps->rd[0], ps->pos[0] + i) & mask;
    const uint32_t c3 = (uint32_t)reader_at(&ps->rd[2], ps->pos[2] + 3 * i) & mask;
    const uint32_t c2 = ((x1 ^ x2 ^ x3) - c1 - c3) & mask;
    out[0][i] = c1;
    out[1][i] = c2;
    out[2][i] = c3;
  }
  ps->pos[0] += n;
  ps->pos[2] += 3 * n;
}

int orc_query(const orc_config* cfg, const uint8_t seeds[48], const uint8_t* db1,
              const uint8_t* db2, const uint8_t* db3, uint64_t s, const uint8_t* q1,
              const uint8_t* q2, const uint8_t* q3, uint32_t persons, int membership,
              const uint64_t* stream_start, orc_out* out) {
  int rc = orc_validate(cfg);
  if (rc) return rc;
  const int be = cfg->backend, var = cfg->variant;
  const unsigned KH = orc_code_bits(var), KMs = orc_mask_bits(var), KC = orc_cmp_bits(var);
  const unsigned KM = KMs ? KMs : 16; /* storage width when shared */
  const int plain = KMs == 0;
  const uint32_t l = cfg->l;
  const uint32_t wl = (l + 63) / 64;
  const uint32_t r = membership ? 1 : cfg->rotations;
  const uint32_t half = (r - 1) / 2;
  const int64_t stride = l / 64;
  const size_t crec = orc_code_record_bytes(be, var, l);
  const size_t rec = crec + orc_mask_record_bytes(be, var, l);
  const uint8_t* dbp[3] = {db1, db2, db3};
  const uint8_t* qp[3] = {q1, q2, q3};
  const uint32_t ncodes = membership ? 1 : 2 * persons;
  const uint64_t ncols = (uint64_t)ncodes * r;
  const uint64_t npairs = membership ? 0 : (uint64_t)persons * (persons ? persons - 1 : 0) / 2 * 4 * r;
  const uint64_t n = ncols * s + npairs;
  const uint64_t W = ceil_div(n, 64);
  const uint32_t mH = kmask(KH), mM = kmask(KM);

  uint32_t lamH[6], lamM[6];
  orc_lambda(KH, lamH);
  orc_lambda(KM, lamM);

  /* ---- dot phase (engine.cpp:304-354), per party ---- */
  uint32_t* hd_add = (uint32_t*)calloc(3 * (n ? n : 1), sizeof(uint32_t));
  uint32_t* ml_add = (uint32_t*)calloc(3 * (n ? n : 1), sizeof(uint32_t));
  int64_t* public_ml = (int64_t*)calloc(n ? n : 1, sizeof(int64_t));
  /* plain masks: the same bits in every party's payload; parse from party 1 */
  uint64_t* qmask = NULL;
  if (plain) {
    qmask = (uint64_t*)calloc((size_t)ncols * wl, sizeof(uint64_t));
    uint64_t* tmp = (uint64_t*)calloc(wl, sizeof(uint64_t));
    for (uint32_t c = 0; c < ncodes; ++c) {
      mask_bits(qp[0] + c * rec + crec, l, tmp);
      for (uint32_t j = 0; j < r; ++j) rotate_bits(tmp, l, ((int64_t)j - (int64_t)half) * stride, qmask + (c * r + j) * wl);
    }
    free(tmp);
#pragma omp parallel for schedule(static)
    for (int64_t row = 0; row < (int64_t)s; ++row) {
      uint64_t dm[256];
      uint64_t* dmw = wl <= 256 ? dm : (uint64_t*)malloc(sizeof(uint64_t) * wl);
      mask_bits(dbp[0] + row * rec + crec, l, dmw);
      for (uint64_t col = 0; col < ncols; ++col) public_ml[col * s + row] = popcount_and(qmask + col * wl, dmw, l);
      if (dmw != dm) free(dmw);
    }
    uint64_t k = ncols * s;
    for (uint32_t i = 0; i < persons && !membership; ++i)
      for (uint32_t j = i + 1; j < persons; ++j)
        for (uint32_t ea = 0; ea < 2; ++ea)
          for (uint32_t eb = 0; eb < 2; ++eb)
            for (uint32_t rot = 0; rot < r; ++rot, ++k)
              public_ml[k] = popcount_and(qmask + ((2 * i + ea) * r + rot) * wl, qmask + ((2 * j + eb) * r + half) * wl, l);
  }
  for (int p = 0; p < 3; ++p) {
    const gr lh = {lamH[2 * p], lamH[2 * p + 1]}, lm = {lamM[2 * p], lamM[2 * p + 1]};
    inst* qc = (inst*)malloc(sizeof(inst) * ncols);
    inst* qm = (inst*)malloc(sizeof(inst) * ncols);
    for (uint32_t c = 0; c < ncodes; ++c) {
      inst code, mask;
      parse_inst(be, qp[p] + c * rec, l, KH, lh, &code);
      if (!plain) parse_inst(be, qp[p] + c * rec + crec, l, KM, lm, &mask);
      for (uint32_t j = 0; j < r; ++j) {
        const int64_t by = ((int64_t)j - (int64_t)half) * stride;
        rotate_inst(be, &code, l, by, &qc[c * r + j]);
        if (!plain) rotate_inst(be, &mask, l, by, &qm[c * r + j]);
      }
      free_inst(&code);
      if (!plain) free_inst(&mask);
    }
#pragma omp parallel for schedule(static)
    for (int64_t row = 0; row < (int64_t)s; ++row) {
      inst dc, dm;
      parse_inst(be, dbp[p] + row * rec, l, KH, lh, &dc);
      if (!plain) parse_inst(be, dbp[p] + row * rec + crec, l, KM, lm, &dm);
      for (uint64_t col = 0; col < ncols; ++col) {
        hd_add[p * n + col * s + row] = dot_row(be, dc.a, dc.b, &qc[col], l, KH);
        if (!plain) ml_add[p * n + col * s + row] = dot_row(be, dm.a, dm.b, &qm[col], l, KM);
      }
      free_inst(&dc);
      if (!plain) free_inst(&dm);
    }
    uint64_t k = 0;
    for (uint32_t i = 0; i < persons && !membership; ++i)
      for (uint32_t j = i + 1; j < persons; ++j)
        for (uint32_t ea = 0; ea < 2; ++ea)
          for (uint32_t eb = 0; eb < 2; ++eb)
            for (uint32_t rot = 0; rot < r; ++rot, ++k) {
              const inst* xs_c = &qc[(2 * i + ea) * r + rot];
              const inst* ys_c = &qc[(2 * j + eb) * r + half];
              hd_add[p * n + ncols * s + k] = dot_row(be, xs_c->a, xs_c->b, ys_c, l, KH);
              if (!plain) {
                const inst* xs_m = &qm[(2 * i + ea) * r + rot];
                const inst* ys_m = &qm[(2 * j + eb) * r + half];
                ml_add[p * n + ncols * s + k] = dot_row(be, xs_m->a, xs_m->b, ys_m, l, KM);
              }
            }
    for (uint64_t c = 0; c < ncols; ++c) {
      free_inst(&qc[c]);
      if (!plain) free_inst(&qm[c]);
    }
    free(qc);
    free(qm);
  }
  free(qmask);
  if (out && out->dot_hd) memcpy(out->dot_hd, hd_add, sizeof(uint32_t) * 3 * n);
  if (out && out->dot_ml) memcpy(out->dot_ml, ml_add, sizeof(uint32_t) * 3 * n);
  if (out && out->public_ml) memcpy(out->public_ml, public_ml, sizeof(int64_t) * n);

  /* ---- PRF streams (A.3) ---- */
  prf_state ps;
  for (int k = 0; k < 3; ++k) {
    ps.seed[k] = seeds + 16 * k;
    reader_init(&ps.rd[k], ps.seed[k]);
    ps.pos[k] = stream_start ? stream_start[k] : 0;
  }

  /* ---- reshare_pair<KH, KM> (engine.cpp:80-106): own = z + F(s_p) - F(s_{p-1}),
   * hd lanes at stream index i, ml lanes (shared masks only) at n + i. ---- */
  const uint64_t nml = plain ? 0 : n;
  uint32_t* hd = (uint32_t*)calloc(3 * (n ? n : 1), sizeof(uint32_t));
  uint32_t* ml = (uint32_t*)calloc(3 * (n ? n : 1), sizeof(uint32_t));
  for (uint64_t i = 0; i < n; ++i) {
    uint32_t fh[3], fm[3] = {0, 0, 0};
    for (int k = 0; k < 3; ++k) fh[k] = (uint32_t)reader_at(&ps.rd[k], ps.pos[k] + i) & mH;
    if (!plain)
      for (int k = 0; k < 3; ++k) fm[k] = (uint32_t)reader_at(&ps.rd[k], ps.pos[k] + n + i) & mM;
    for (int p = 0; p < 3; ++p) {
      const int q = (p + 2) % 3;
      hd[p * n + i] = (hd_add[p * n + i] + fh[p] - fh[q]) & mH;
      ml[p * n + i] = plain ? 0 : ((ml_add[p * n + i] + fm[p] - fm[q]) & mM);
    }
  }
  for (int k = 0; k < 3; ++k) ps.pos[k] += n + nml;
  if (out && out->rs_hd) memcpy(out->rs_hd, hd, sizeof(uint32_t) * 3 * n);
  if (out && out->rs_ml) memcpy(out->rs_ml, ml, sizeof(uint32_t) * 3 * n);

  /* ---- comparison input ---- */
  uint32_t* ml32 = (uint32_t*)calloc(3 * (n ? n : 1), sizeof(uint32_t));
  uint32_t* diff = (uint32_t*)calloc(3 * (n ? n : 1), sizeof(uint32_t));
  uint64_t lift_gates = 0;
  if (plain) {
    /* plain_diff_lanes<16> (engine.hpp:77-90): public_minus(ceil((1-2r) ml), hd):
     * component 1 absorbs the public constant (rep3.hpp:59-65). */
    for (uint64_t i = 0; i < n; ++i) {
      const int64_t t = (int64_t)ceil((1.0 - 2.0 * cfg->ratio) * (double)public_ml[i]);
      diff[i] = ((uint32_t)(uint64_t)t - hd[i]) & 0xFFFFu;
      diff[n + i] = (0u - hd[n + i]) & 0xFFFFu;
      diff[2 * n + i] = (0u - hd[2 * n + i]) & 0xFFFFu;
    }
  } else {
    if (KMs == 16) {
      /* ---- lift<16,16> (convert.hpp:169-192) ---- */
      const uint32_t* mlc[3] = {ml, ml + n, ml + 2 * n};
      uint64_t*** xs = share_split(mlc, n, W, 16);
      const unsigned lidx[2] = {16, 17};
      brow ext[2] = {brow_new(W), brow_new(W)};
      bit_extract(&ps, n, W, 16, (uint64_t* const**)xs, lidx, 2, ext);
      free_split(xs, 16);
      lift_gates = 64;
      uint32_t* inj17 = (uint32_t*)malloc(sizeof(uint32_t) * 3 * (n ? n : 1));
      uint32_t* inj16 = (uint32_t*)malloc(sizeof(uint32_t) * 3 * (n ? n : 1));
      uint32_t* i17[3] = {inj17, inj17 + n, inj17 + 2 * n};
      uint32_t* i16[3] = {inj16, inj16 + n, inj16 + 2 * n};
      bit_inject(&ps, &ext[1], n, 15, i17); /* bit K+1 into Z_2^(M-1) first */
      bit_inject(&ps, &ext[0], n, 16, i16);
      brow_free(&ext[0]);
      brow_free(&ext[1]);
      for (uint64_t i = 0; i < 3 * n; ++i) ml32[i] = ml[i] - (inj17[i] << 17) - (inj16[i] << 16);
      free(inj17);
      free(inj16);
    } else {
      memcpy(ml32, ml, sizeof(uint32_t) * 3 * n); /* KM = 32: already wide */
    }
    /* shared_diff_lanes (engine.hpp:94-120): a*ml32 - b*hd (const_lift for KH=16,
     * mul_public for KH=32: the same product in Z_2^32) */
    for (uint64_t i = 0; i < 3 * n; ++i) diff[i] = cfg->a * ml32[i] - cfg->b * hd[i];
  }
  if (out && out->ml32) memcpy(out->ml32, ml32, sizeof(uint32_t) * 3 * n);
  if (out && out->diff) memcpy(out->diff, diff, sizeof(uint32_t) * 3 * n);

  /* ---- msb_batch<KC> (circuits.hpp:300-306) ---- */
  const uint32_t* dc[3] = {diff, diff + n, diff + 2 * n};
  uint64_t*** xs = share_split(dc, n, W, KC);
  const unsigned midx[1] = {KC - 1};
  brow bits = brow_new(W);
  bit_extract(&ps, n, W, KC, (uint64_t* const**)xs, midx, 1, &bits);
  free_split(xs, KC);
  if (out && out->msb)
    for (int p = 0; p < 3; ++p)
      for (uint64_t i = 0; i < n; ++i) out->msb[p * n + i] = (bits.c[p][i / 64] >> (i % 64)) & 1;
  if (out && out->row_bits && cfg->debug_rows)
    for (uint64_t i = 0; i < n; ++i)
      out->row_bits[i] =
          ((bits.c[0][i / 64] ^ bits.c[1][i / 64] ^ bits.c[2][i / 64]) >> (i % 64)) & 1;

  /* ---- aggregation: groups + or_tree_batch (engine.cpp:376-387,
   * circuits.hpp:387-434) ---- */
  const uint32_t ngroups = membership ? 1 : persons;
  uint64_t* glen = (uint64_t*)calloc(ngroups ? ngroups : 1, sizeof(uint64_t));
  uint64_t** glanes = (uint64_t**)calloc(ngroups ? ngroups : 1, sizeof(uint64_t*));
  for (uint32_t g = 0; g < ngroups; ++g) {
    const uint64_t cnt = membership ? s : 2ull * r * s + (uint64_t)(persons - 1) * 4 * r;
    glanes[g] = (uint64_t*)malloc(sizeof(uint64_t) * (cnt ? cnt : 1));
  }
  if (membership) {
    for (uint64_t i = 0; i < s; ++i) glanes[0][glen[0]++] = i;
  } else {
    for (uint64_t c = 0; c < ncodes; ++c)
      for (uint32_t j = 0; j < r; ++j) {
        const uint64_t base = (c * r + j) * s;
        for (uint64_t row = 0; row < s; ++row) glanes[c / 2][glen[c / 2]++] = base + row;
      }
    uint64_t k = ncols * s;
    for (uint32_t i = 0; i < persons; ++i)
      for (uint32_t j = i + 1; j < persons; ++j)
        for (uint32_t e = 0; e < 4 * r; ++e, ++k) {
          glanes[i][glen[i]++] = k;
          glanes[j][glen[j]++] = k;
        }
  }
  brow* grp = (brow*)malloc(sizeof(brow) * (ngroups ? ngroups : 1));
  uint64_t* gl = (uint64_t*)malloc(sizeof(uint64_t) * (ngroups ? ngroups : 1));
  for (uint32_t g = 0; g < ngroups; ++g) {
    gl[g] = glen[g];
    grp[g] = brow_new(ceil_div(glen[g], 64));
    for (uint64_t i = 0; i < glen[g]; ++i) {
      const uint64_t ln = glanes[g][i];
      for (int p = 0; p < 3; ++p)
        if ((bits.c[p][ln / 64] >> (ln % 64)) & 1) grp[g].c[p][i / 64] |= (uint64_t)1 << (i % 64);
    }
  }
  uint64_t or_rounds = 0, or_bytes = 0;
  or_tree_groups(&ps, grp, gl, ngroups, &or_rounds, &or_bytes);
  /* open_bits_to(agg, P1) (circuits.hpp:449-486) */
  if (out && out->person_match)
    for (uint32_t g = 0; g < ngroups; ++g)
      out->person_match[g] =
          gl[g] == 0 ? 0 : (uint8_t)((grp[g].c[0][0] ^ grp[g].c[1][0] ^ grp[g].c[2][0]) & 1);
  if (out && out->agg)
    for (uint32_t g = 0; g < ngroups; ++g)
      for (int p = 0; p < 3; ++p) out->agg[p * ngroups + g] = gl[g] == 0 ? 0 : (uint8_t)(grp[g].c[p][0] & 1);
  if (out && out->stream_pos)
    for (int k = 0; k < 3; ++k) out->stream_pos[k] = ps.pos[k];

  /* analytic ledger (A.5) */
  if (out && out->stats) {
    const uint64_t nb8 = ceil_div(n, 8);
    const uint64_t open_bytes = ceil_div(ngroups, 8);
    const uint64_t msb_gates = 2 * KC - 3;
    for (int p = 0; p < 3; ++p) {
      orc_stats* st = &out->stats[p];
      st->dot_bytes = n * (KH / 8) + nml * (KM / 8);
      st->dot_rounds = 1;
      const uint64_t ot = lift_gates ? ((p == 0) ? 8 * n : 4 * n) : 0;
      st->lift_bytes = lift_gates * nb8 + ot;
      st->lift_rounds = lift_gates ? 17 + 4 : 0;
      st->msb_bytes = msb_gates * nb8;
      st->msb_rounds = KC - 1;
      st->or_tree_bytes = or_bytes + (p == 0 ? 0 : open_bytes) + (cfg->debug_rows && p != 0 ? nb8 : 0);
      st->or_tree_rounds = or_rounds + 1 + (cfg->debug_rows ? 1 : 0);
    }
  }

  for (uint32_t g = 0; g < ngroups; ++g) {
    free(glanes[g]);
    brow_free(&grp[g]);
  }
  free(glanes);
  free(glen);
  free(grp);
  free(gl);
  brow_free(&bits);
  free(hd_add);
  free(ml_add);
  free(public_ml);
  free(hd);
  free(ml);
  free(ml32);
  free(diff);
  return 0;
}

int orc_run_local(const orc_config* cfg, uint64_t seed, uint64_t s, const uint64_t* db_codes,
                  const uint64_t* db_masks, uint32_t persons, const uint64_t* q_codes,
                  const uint64_t* q_masks, int membership, orc_out* out) {
  int rc = orc_validate(cfg);
  if (rc) return rc;
  const size_t rec = orc_code_record_bytes(cfg->backend, cfg->variant, cfg->l) +
                     orc_mask_record_bytes(cfg->backend, cfg->variant, cfg->l);
  const uint32_t ncodes = membership ? 1 : 2 * persons;
  uint8_t* db[3];
  uint8_t* q[3];
  for (int p = 0; p < 3; ++p) {
    db[p] = (uint8_t*)malloc(rec * (s ? s : 1));
    q[p] = (uint8_t*)malloc(rec * (ncodes ? ncodes : 1));
  }
  orc_rng* dr = orc_rng_sub(seed, 1);
  orc_rng* qr = orc_rng_sub(seed, 2);
  orc_deal_payload_v(cfg->backend, cfg->variant, cfg->l, s, db_codes, db_masks, dr, db[0], db[1], db[2]);
  orc_deal_payload_v(cfg->backend, cfg->variant, cfg->l, ncodes, q_codes, q_masks, qr, q[0], q[1], q[2]);
  orc_rng_free(dr);
  orc_rng_free(qr);
  uint8_t seeds[48];
  orc_party_seeds(seed, seeds);
  rc = orc_query(cfg, seeds, db[0], db[1], db[2], s, q[0], q[1], q[2], persons, membership, NULL, out);
  for (int p = 0; p < 3; ++p) {
    free(db[p]);
    free(q[p]);
  }
  return rc;
}
