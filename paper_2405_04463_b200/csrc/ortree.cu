// K5 (share-exact): the reference's halving OR tree over each person's lanes,
// or_tree_batch (include/irismpc/circuits.hpp:387-434) with and_layer's AND
// gates (circuits.hpp:92-131) and the reference's PRF draws (SURVEY.md A.3:
// per level, per group in order, one gate of nb lanes = ceil(nb/64) words of
// every seed stream, right after the msb gates).  So the aggregate shares
// equal the reference's share for share, not only the opened bit.
//
// Groups (Schedule::groups, src/engine.cpp:221-289): group g lists its DB lanes
// (codes 2g, 2g+1, all rotations, all rows: one contiguous lane range) then its
// inner-batch pair lanes (pairs (i, g), i < g, then (g, j), j > g, 4r lanes
// each); membership / comparison: one group of every lane.  Level t folds a row
// of N lanes into na = ceil(N/2): lo = lanes [0, na), hi = lanes [na, N),
// out = lo ^ hi ^ AND(lo, hi) with the AND masked to nb = N - na lanes.
//
// Layout: level 0 reads the lane bits in reference lane order (the msb
// kernels' match words, 64-lane little-endian words); every level writes
// compact rows [comp][group][ceil(na/64)] into one of two ping-pong buffers.
// Thread = 8 consecutive output words of one group: 2 ChaCha12 blocks per seed
// cover its 8 gate words.
#include "common.cuh"
#include "kernels.h"

namespace irisgpu {

namespace {

__device__ __forceinline__ uint64_t funnel(const uint64_t* w, uint64_t bit) {
  const uint64_t i = bit / 64;
  const int sh = (int)(bit % 64);
  return sh ? (w[i] >> sh) | (w[i + 1] << (64 - sh)) : w[i];
}

__device__ __forceinline__ uint64_t lane_mask(int64_t live) {
  return live >= 64 ? ~0ull : (live <= 0 ? 0ull : (1ull << live) - 1);
}

// global lane of position i of group g's lane list
__device__ __forceinline__ uint64_t group_lane(const OrTreeArgs& A, uint32_t g, uint64_t i) {
  if (i < A.db_lanes) return (uint64_t)g * A.db_lanes + i;
  const uint64_t q = (i - A.db_lanes) / A.pair_block, o = (i - A.db_lanes) % A.pair_block;
  const uint32_t a = q < g ? (uint32_t)q : g, b = q < g ? g : (uint32_t)q + 1;
  const uint64_t pidx = (uint64_t)a * A.ngroups - (uint64_t)a * (a + 1) / 2 + (b - a - 1);
  return A.pair_base + pidx * A.pair_block + o;
}

// 64 list positions [i, i + 64) of group g, component c, from the lane bits
// (positions >= lanes read as 0 or garbage; the callers mask them)
__device__ __forceinline__ uint64_t list64(const OrTreeArgs& A, int c, uint32_t g, uint64_t i) {
  const uint64_t* m = A.match[c];
  if (i + 64 <= A.db_lanes) return funnel(m, (uint64_t)g * A.db_lanes + i);
  if (i >= A.db_lanes && A.pair_block) {
    const uint64_t o = (i - A.db_lanes) % A.pair_block;
    if (o + 64 <= A.pair_block) return funnel(m, group_lane(A, g, i));
  }
  uint64_t v = 0;
  for (int b = 0; b < 64; ++b) {
    const uint64_t pos = i + b;
    if (pos >= A.lanes) break;
    const uint64_t ln = group_lane(A, g, pos);
    v |= ((m[ln / 64] >> (ln % 64)) & 1ull) << b;
  }
  return v;
}

// Output word wi of group g at level L, given its gate words f[seed] (used
// when wi < ceil(nb/64)).  L0: the source is the lane bits via the group
// lists; else the previous level's compact rows (stride win, row gi).  Output
// row go (stride wo).
template <bool L0>
__device__ __forceinline__ void fold_word(const OrTreeArgs& A, const OrTreeLevel& L, uint32_t g, uint64_t wi,
                                          uint64_t gi, uint64_t go, const uint64_t f[3]) {
  const uint64_t nbw = (L.nb + 63) / 64;
  const uint64_t ml = lane_mask((int64_t)L.na - 64 * (int64_t)wi);
  const uint64_t mh = lane_mask((int64_t)L.nb - 64 * (int64_t)wi);
  uint64_t lo[3], hi[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    if (L0) {
      lo[c] = list64(A, c, g, 64 * wi) & ml;
      hi[c] = mh ? list64(A, c, g, L.na + 64 * wi) & mh : 0ull;
    } else {
      const uint64_t* row = L.in[c] + gi * L.win;
      lo[c] = row[wi] & ml;
      hi[c] = mh ? funnel(row, L.na + 64 * wi) & mh : 0ull;
    }
  }
  uint64_t z[3] = {0, 0, 0};
  if (wi < nbw) {
    // z_p = x_p y_p ^ x_{p-1} y_p ^ x_p y_{p-1} ^ F_p ^ F_{p-1}, dead lanes zeroed (mask_lanes)
#pragma unroll
    for (int p = 0; p < 3; ++p) {
      const int q = (p + 2) % 3;
      z[p] = ((lo[p] & hi[p]) ^ (lo[q] & hi[p]) ^ (lo[p] & hi[q]) ^ f[p] ^ f[q]) & mh;
    }
  }
#pragma unroll
  for (int c = 0; c < 3; ++c) L.out[c][go * L.wo + wi] = lo[c] ^ hi[c] ^ z[c];
}

// Output words w0 .. w0 + 7 of group g at level L, their gate words computed
// here: 2 ChaCha12 blocks per seed cover the 8 stream elements.
template <bool L0>
__device__ __forceinline__ void level_words(const OrTreeArgs& A, const OrTreeLevel& L, uint32_t g, uint64_t w0) {
  const uint64_t wout = (L.na + 63) / 64;
  const uint64_t nbw = (L.nb + 63) / 64;
  uint64_t f[3][8];
  if (w0 < nbw) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const uint64_t e0 = L.rand_base[k] + (uint64_t)g * nbw + w0;
      const int r = (int)(e0 % 8);
      uint64_t x[16];  // elements 8 (e0 / 8) .. + 15: word w of the window is x[w + r]
      uint32_t blk[16];
      chacha12_block(A.key[k], e0 / 8, 0, blk);
#pragma unroll
      for (int w = 0; w < 8; ++w) x[w] = chacha_word(blk, w);
      if (r) {
        chacha12_block(A.key[k], e0 / 8 + 1, 0, blk);
#pragma unroll
        for (int w = 0; w < 8; ++w) x[8 + w] = chacha_word(blk, w);
      }
      // static-index select of x[w + r] (a runtime index would put x in local memory)
#pragma unroll
      for (int w = 0; w < 8; ++w) {
        uint64_t v = x[w];
#pragma unroll
        for (int q = 1; q < 8; ++q)
          if (r == q) v = x[w + q];
        f[k][w] = v;
      }
    }
  }
#pragma unroll
  for (int w = 0; w < 8; ++w) {
    if (w0 + w < wout) {
      const uint64_t fw[3] = {f[0][w], f[1][w], f[2][w]};
      fold_word<L0>(A, L, g, w0 + w, g, g, fw);
    }
  }
}

}  // namespace

// One level of every group, thread = 8 output words of one group.
template <bool L0>
__global__ void __launch_bounds__(128) k_ortree_level(const __grid_constant__ OrTreeArgs A, OrTreeLevel L) {
  const uint64_t per = ((L.na + 63) / 64 + 7) / 8;
  const uint64_t id = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (id >= (uint64_t)A.ngroups * per) return;
  level_words<L0>(A, L, (uint32_t)(id / per), (id % per) * 8);
}

namespace {
constexpr uint64_t kTailWords = 480;  // a row of at most this many output words runs in k_ortree_tail
constexpr int kTailThreads = 256;
constexpr int kTailRand = 2 * kTailWords + 24;  // gate words of all tail levels, per seed
constexpr int kTailLevels = 24;
}  // namespace

// The remaining levels once a group's row is at most kTailWords words: CTA =
// group.  First every gate word of every remaining level (they do not depend
// on the data) is drawn in parallel, one ChaCha12 block per thread per step,
// into shared memory; then the levels run back to back on shared-memory rows
// (ping-pong), separated by __syncthreads, and lane 0 -> out[comp][group].  L
// is the first of these levels, reading the global rows (or the lane bits);
// its rand_base is group 0's, every level advances it by ngroups x ceil(nb/64).
template <bool L0>
__global__ void __launch_bounds__(kTailThreads) k_ortree_tail(const __grid_constant__ OrTreeArgs A, OrTreeLevel L,
                                                              uint8_t* out) {
  __shared__ uint64_t rows[2][3][kTailWords + 8];
  __shared__ uint64_t rnd[3][kTailRand];
  const uint32_t g = blockIdx.x;
  // the levels' gate ranges: level t draws nbw_t words at base_t + g * nbw_t
  __shared__ uint32_t lvl_off[kTailLevels + 1], lvl_nbw[kTailLevels], first[kTailLevels + 1];
  __shared__ uint64_t lvl_e0[kTailLevels][3];
  __shared__ int nl_s;
  if (threadIdx.x == 0) {
    uint64_t N = L.na + L.nb, base[3] = {L.rand_base[0], L.rand_base[1], L.rand_base[2]};
    uint32_t off = 0, jobs = 0;
    int nl = 0;
    while (N > 1 && nl < kTailLevels) {
      const uint64_t na = (N + 1) / 2, nbw = (N - na + 63) / 64;
      lvl_off[nl] = off;
      lvl_nbw[nl] = (uint32_t)nbw;
      first[nl] = jobs;
      for (int k = 0; k < 3; ++k) {
        lvl_e0[nl][k] = base[k] + (uint64_t)g * nbw;
        base[k] += (uint64_t)A.ngroups * nbw;
        jobs += (uint32_t)((lvl_e0[nl][k] + nbw - 1) / 8 - lvl_e0[nl][k] / 8 + 1);
      }
      off += (uint32_t)nbw;
      N = na;
      ++nl;
    }
    lvl_off[nl] = off;
    first[nl] = jobs;
    nl_s = nl;
  }
  __syncthreads();
  const int nl = nl_s;
  // ChaCha blocks: per (level, seed), the blocks covering [e0, e0 + nbw)
  for (uint32_t j = threadIdx.x; j < first[nl]; j += blockDim.x) {
    int t = 0;
    while (first[t + 1] <= j) ++t;
    uint32_t r = j - first[t];
    int k = 0;
    for (; k < 2; ++k) {
      const uint32_t nbk = (uint32_t)((lvl_e0[t][k] + lvl_nbw[t] - 1) / 8 - lvl_e0[t][k] / 8 + 1);
      if (r < nbk) break;
      r -= nbk;
    }
    const uint64_t e0 = lvl_e0[t][k], b = e0 / 8 + r;
    uint32_t blk[16];
    chacha12_block(A.key[k], b, 0, blk);
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      const uint64_t e = b * 8 + w;
      if (e >= e0 && e < e0 + lvl_nbw[t]) rnd[k][lvl_off[t] + (e - e0)] = chacha_word(blk, w);
    }
  }
  __syncthreads();
  int cur = -1;  // -1: the global input of the first level
  for (int t = 0; t < nl; ++t) {
    const int nxt = cur == 0 ? 1 : 0;
    for (int c = 0; c < 3; ++c) L.out[c] = rows[nxt][c];
    const uint64_t wout = (L.na + 63) / 64;
    for (uint64_t wi = threadIdx.x; wi < wout; wi += blockDim.x) {
      const uint64_t f[3] = {wi < lvl_nbw[t] ? rnd[0][lvl_off[t] + wi] : 0ull,
                             wi < lvl_nbw[t] ? rnd[1][lvl_off[t] + wi] : 0ull,
                             wi < lvl_nbw[t] ? rnd[2][lvl_off[t] + wi] : 0ull};
      if (cur < 0)
        fold_word<L0>(A, L, g, wi, g, 0, f);
      else
        fold_word<false>(A, L, g, wi, 0, 0, f);
    }
    __syncthreads();
    const uint64_t N = L.na;
    cur = nxt;
    L.na = (N + 1) / 2;
    L.nb = N - L.na;
    L.win = L.wo;
    L.wo = (L.na + 63) / 64;
    for (int c = 0; c < 3; ++c) L.in[c] = rows[cur][c];
  }
  if (threadIdx.x == 0)
    for (int c = 0; c < 3; ++c) {
      uint64_t v;
      if (cur >= 0)
        v = rows[cur][c][0];
      else if (L0)
        v = list64(A, c, g, 0);
      else
        v = L.in[c][(uint64_t)g * L.win];
      out[(uint64_t)c * A.ngroups + g] = A.lanes ? (uint8_t)(v & 1ull) : 0;
    }
}

uint64_t ortree_scratch_words(uint32_t ngroups, uint64_t lanes) {
  const uint64_t na = (lanes + 1) / 2;
  return 3ull * ngroups * ((na + 63) / 64) + 8;
}

int launch_ortree(const OrTreeArgs& a, const uint64_t rand_start[3], uint64_t* scratch[2], uint8_t* out,
                  cudaStream_t st) {
  if (!a.ngroups) return 0;
  int launches = 0;
  uint64_t N = a.lanes, win = 0, base[3] = {rand_start[0], rand_start[1], rand_start[2]};
  int cur = -1;  // -1: the lane bits
  const uint64_t comp_stride = ortree_scratch_words(a.ngroups, a.lanes) / 3;
  while (true) {
    OrTreeLevel L{};
    L.na = (N + 1) / 2;
    L.nb = N - L.na;
    L.wo = (L.na + 63) / 64;
    L.win = win;
    const int nxt = cur == 0 ? 1 : 0;
    for (int c = 0; c < 3; ++c) {
      L.out[c] = scratch[nxt] + c * comp_stride;
      L.in[c] = cur < 0 ? nullptr : scratch[cur] + c * comp_stride;
    }
    for (int k = 0; k < 3; ++k) L.rand_base[k] = base[k];
    if (N <= 1 || L.wo <= kTailWords) {  // the rest (possibly no level at all) in one launch
      if (cur < 0)
        k_ortree_tail<true><<<a.ngroups, kTailThreads, 0, st>>>(a, L, out);
      else
        k_ortree_tail<false><<<a.ngroups, kTailThreads, 0, st>>>(a, L, out);
      return launches + 1;
    }
    const uint64_t threads = (uint64_t)a.ngroups * ((L.wo + 7) / 8);
    const unsigned blocks = (unsigned)((threads + 127) / 128);
    if (cur < 0)
      k_ortree_level<true><<<blocks, 128, 0, st>>>(a, L);
    else
      k_ortree_level<false><<<blocks, 128, 0, st>>>(a, L);
    ++launches;
    const uint64_t nbw = (L.nb + 63) / 64;
    for (int k = 0; k < 3; ++k) base[k] += (uint64_t)a.ngroups * nbw;
    N = L.na;
    win = L.wo;
    cur = nxt;
  }
}

}  // namespace irisgpu
