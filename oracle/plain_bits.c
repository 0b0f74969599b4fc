/* Plaintext per-lane match bits at full scale -- TEST INFRASTRUCTURE ONLY.
 *
 * The reference test oracle (/root/reference/proj/tests/oracle.hpp:35-57):
 * for a (query, DB row) pair, ml = popcount(q.mask & db.mask) and
 * hd = popcount((q.code ^ db.code) & q.mask & db.mask); the masked dot is
 * ml - 2 hd (iris.hpp:108-112) and the predicate is
 *   shared masks:  b * (ml - 2 hd) > a * ml
 *   public masks:  (ml - 2 hd) > ceil((1 - 2 ratio) * ml)
 * evaluated over the lane schedule of Session::batch_query
 * (src/engine.cpp:262-293): DB lanes (c * r + j) * s + row, the query code c
 * rotated by (j - (r-1)/2) * (l/64) bits (rotate_vec, engine.hpp:126-136:
 * element i moves to (i + off) mod l), then the inner-batch pair lanes in
 * (i < j, ea, eb, rot) order, rotated eye of person i vs the unrotated eye of
 * person j.  Person bits are the OR over each person's lanes.
 *
 * No MPC, no shares: it is the independent plaintext check of the GPU's
 * opened per-lane bits (debug_rows) at BASELINE sizes (up to 2e9 lanes), so it
 * is plain C + OpenMP, compiled with -O3 -march=native on the machine that
 * runs it (tests/test_full_scale.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static int pred(int64_t ml, int64_t hd, int public_mask, double ratio, uint32_t a, uint32_t b) {
  const int64_t dot = ml - 2 * hd;
  if (public_mask) return dot > (int64_t)ceil((1.0 - 2.0 * ratio) * (double)ml);
  return (int64_t)b * dot > (int64_t)a * ml;
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

#if defined(__AVX512F__) && defined(__AVX512VPOPCNTDQ__)
#include <immintrin.h>
static inline void counts(const uint64_t* qc, const uint64_t* qm, const uint64_t* dc, const uint64_t* dm,
                          uint32_t wl, int64_t* ml, int64_t* hd) {
  __m512i m = _mm512_setzero_si512(), h = _mm512_setzero_si512();
  uint32_t w = 0;
  for (; w + 8 <= wl; w += 8) {
    const __m512i mm = _mm512_and_si512(_mm512_loadu_si512(qm + w), _mm512_loadu_si512(dm + w));
    const __m512i x = _mm512_and_si512(_mm512_xor_si512(_mm512_loadu_si512(qc + w), _mm512_loadu_si512(dc + w)), mm);
    m = _mm512_add_epi64(m, _mm512_popcnt_epi64(mm));
    h = _mm512_add_epi64(h, _mm512_popcnt_epi64(x));
  }
  int64_t mt = _mm512_reduce_add_epi64(m), ht = _mm512_reduce_add_epi64(h);
  for (; w < wl; ++w) {
    const uint64_t mm = qm[w] & dm[w];
    mt += __builtin_popcountll(mm);
    ht += __builtin_popcountll((qc[w] ^ dc[w]) & mm);
  }
  *ml = mt;
  *hd = ht;
}
/* four query columns against one DB row: the DB vectors are loaded once */
static inline void counts4(const uint64_t* const qc[4], const uint64_t* const qm[4], const uint64_t* dc,
                           const uint64_t* dm, uint32_t wl, int64_t ml[4], int64_t hd[4]) {
  __m512i m[4], h[4];
  for (int c = 0; c < 4; ++c) m[c] = h[c] = _mm512_setzero_si512();
  uint32_t w = 0;
  for (; w + 8 <= wl; w += 8) {
    const __m512i d_m = _mm512_loadu_si512(dm + w), d_c = _mm512_loadu_si512(dc + w);
    for (int c = 0; c < 4; ++c) {
      const __m512i mm = _mm512_and_si512(_mm512_loadu_si512(qm[c] + w), d_m);
      const __m512i x = _mm512_and_si512(_mm512_xor_si512(_mm512_loadu_si512(qc[c] + w), d_c), mm);
      m[c] = _mm512_add_epi64(m[c], _mm512_popcnt_epi64(mm));
      h[c] = _mm512_add_epi64(h[c], _mm512_popcnt_epi64(x));
    }
  }
  for (int c = 0; c < 4; ++c) {
    int64_t mt = _mm512_reduce_add_epi64(m[c]), ht = _mm512_reduce_add_epi64(h[c]);
    for (uint32_t v = w; v < wl; ++v) {
      const uint64_t mm = qm[c][v] & dm[v];
      mt += __builtin_popcountll(mm);
      ht += __builtin_popcountll((qc[c][v] ^ dc[v]) & mm);
    }
    ml[c] = mt;
    hd[c] = ht;
  }
}
#define HAVE_COUNTS4 1
#else
static inline void counts(const uint64_t* qc, const uint64_t* qm, const uint64_t* dc, const uint64_t* dm,
                          uint32_t wl, int64_t* ml, int64_t* hd) {
  int64_t m = 0, h = 0;
  for (uint32_t w = 0; w < wl; ++w) {
    const uint64_t mm = qm[w] & dm[w];
    m += __builtin_popcountll(mm);
    h += __builtin_popcountll((qc[w] ^ dc[w]) & mm);
  }
  *ml = m;
  *hd = h;
}
#endif

/* Lanes of a batch query (membership: one code, r = 1, s lanes, one group).
 * lane_bits [n] (may be NULL) receives the plaintext bits; if `expect` [n] is
 * given, mismatching lanes are counted (first one in *first_bad).  person
 * [persons] receives the per-person OR.  Returns the number of mismatches. */
uint64_t plain_batch_bits(uint32_t l, uint32_t r, int membership, int public_mask, double ratio, uint32_t a,
                          uint32_t b, uint64_t s, const uint64_t* db_codes, const uint64_t* db_masks,
                          uint32_t persons, const uint64_t* q_codes, const uint64_t* q_masks, uint8_t* lane_bits,
                          const uint8_t* expect, uint64_t* first_bad, uint8_t* person) {
  const uint32_t wl = (l + 63) / 64;
  const uint32_t ncodes = membership ? 1u : 2u * persons;
  const uint32_t rr = membership ? 1u : r;
  const uint32_t half = (rr - 1) / 2;
  const int64_t stride = l / 64;
  const uint64_t ncols = (uint64_t)ncodes * rr;
  uint64_t* rq_c = (uint64_t*)malloc(sizeof(uint64_t) * wl * (ncols ? ncols : 1));
  uint64_t* rq_m = (uint64_t*)malloc(sizeof(uint64_t) * wl * (ncols ? ncols : 1));
  for (uint32_t c = 0; c < ncodes; ++c)
    for (uint32_t j = 0; j < rr; ++j) {
      const int64_t by = ((int64_t)j - (int64_t)half) * stride;
      rotate_bits(q_codes + (uint64_t)c * wl, l, by, rq_c + ((uint64_t)c * rr + j) * wl);
      rotate_bits(q_masks + (uint64_t)c * wl, l, by, rq_m + ((uint64_t)c * rr + j) * wl);
    }
  const uint32_t ngroups = membership ? 1u : persons;
  uint64_t bad = 0, fb = UINT64_MAX;
  uint8_t* pbits = (uint8_t*)calloc(ngroups ? ngroups : 1, 1);
  const uint64_t RB = 32; /* DB rows per tile: reused across every query column */
  const int64_t ntiles = (int64_t)((s + RB - 1) / RB);
#pragma omp parallel
  {
    uint8_t* mine = (uint8_t*)calloc(ngroups ? ngroups : 1, 1);
    uint64_t my_bad = 0, my_fb = UINT64_MAX;
#pragma omp for schedule(dynamic, 4)
    for (int64_t t = 0; t < ntiles; ++t) {
      const uint64_t r0 = (uint64_t)t * RB, r1 = r0 + RB < s ? r0 + RB : s;
      uint64_t col = 0;
#ifdef HAVE_COUNTS4
      for (; col + 4 <= ncols; col += 4) {
        const uint64_t* qc4[4];
        const uint64_t* qm4[4];
        for (int c = 0; c < 4; ++c) {
          qc4[c] = rq_c + (col + c) * wl;
          qm4[c] = rq_m + (col + c) * wl;
        }
        for (uint64_t row = r0; row < r1; ++row) {
          int64_t ml[4], hd[4];
          counts4(qc4, qm4, db_codes + row * wl, db_masks + row * wl, wl, ml, hd);
          for (int c = 0; c < 4; ++c) {
            const uint8_t bit = (uint8_t)pred(ml[c], hd[c], public_mask, ratio, a, b);
            const uint64_t lane = (col + c) * s + row;
            if (lane_bits) lane_bits[lane] = bit;
            if (expect && expect[lane] != bit) {
              ++my_bad;
              if (lane < my_fb) my_fb = lane;
            }
            mine[membership ? 0u : (uint32_t)((col + c) / rr / 2)] |= bit;
          }
        }
      }
#endif
      for (; col < ncols; ++col) {
        const uint64_t* qc = rq_c + col * wl;
        const uint64_t* qm = rq_m + col * wl;
        const uint32_t g = membership ? 0u : (uint32_t)(col / rr / 2);
        uint8_t any = 0;
        for (uint64_t row = r0; row < r1; ++row) {
          int64_t ml, hd;
          counts(qc, qm, db_codes + row * wl, db_masks + row * wl, wl, &ml, &hd);
          const uint8_t bit = (uint8_t)pred(ml, hd, public_mask, ratio, a, b);
          const uint64_t lane = col * s + row;
          if (lane_bits) lane_bits[lane] = bit;
          if (expect && expect[lane] != bit) {
            ++my_bad;
            if (lane < my_fb) my_fb = lane;
          }
          any |= bit;
        }
        mine[g] |= any;
      }
    }
#pragma omp critical
    {
      for (uint32_t g = 0; g < ngroups; ++g) pbits[g] |= mine[g];
      bad += my_bad;
      if (my_fb < fb) fb = my_fb;
    }
    free(mine);
  }
  /* inner-batch pair lanes (serial: at most persons^2 * 4 * r lanes) */
  if (!membership) {
    uint64_t k = ncols * s;
    for (uint32_t i = 0; i < persons; ++i)
      for (uint32_t j = i + 1; j < persons; ++j)
        for (uint32_t ea = 0; ea < 2; ++ea)
          for (uint32_t eb = 0; eb < 2; ++eb)
            for (uint32_t rot = 0; rot < rr; ++rot, ++k) {
              int64_t ml, hd;
              const uint64_t x = (uint64_t)(2 * i + ea) * rr + rot, y = (uint64_t)(2 * j + eb) * rr + half;
              counts(rq_c + x * wl, rq_m + x * wl, rq_c + y * wl, rq_m + y * wl, wl, &ml, &hd);
              const uint8_t bit = (uint8_t)pred(ml, hd, public_mask, ratio, a, b);
              if (lane_bits) lane_bits[k] = bit;
              if (expect && expect[k] != bit) {
                ++bad;
                if (k < fb) fb = k;
              }
              pbits[i] |= bit;
              pbits[j] |= bit;
            }
  }
  if (person) memcpy(person, pbits, ngroups);
  if (first_bad) *first_bad = fb;
  free(pbits);
  free(rq_c);
  free(rq_m);
  return bad;
}
