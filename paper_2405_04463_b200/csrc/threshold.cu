// K4: the mpc-lift threshold comparison for all three parties, as a pipeline
// of kernels over a lane chunk (one segment per DB column, or the pair lanes).
//
// Replaces, per lane, reshare_pair<16,16> (src/engine.cpp:80-106),
// lift<16,16> = share_split + bit_extract_sum{16,17} + bit_inject<15>,<16>
// (include/irismpc/convert.hpp:84-192, circuits.hpp:152-296),
// shared_diff_lanes<16,16> (engine.hpp:94-120) and msb_batch<32>
// (circuits.hpp:300-306).  The three parties live in one GPU, so a sharing is
// held as its three components and every exchange is a register read.
//
// PRF draws follow the reference stream layout exactly, so
// every intermediate share equals the reference's: for n lanes, W = ceil(n/64)
// words and per-seed query start pos_k:
//   reshare hd lane i -> pos + i,  ml -> pos + n + i
//   lift AND gate g (0..63), 64-lane word w -> pos + 2n + g W + w
//   inject<15>: seed1 c1 -> pos1 + 2n + 64W + i, seed3 c3 -> pos3 + 2n + 64W + 3i
//   (comparison-only, party_comparison_only: no reshare, every offset 2n smaller)
//   inject<16>: seed1 -> pos1 + 3n + 64W + i,    seed3 -> pos3 + 5n + 64W + 3i
//   msb gate g (0..60): seed1 pos1 + 4n + 64W + gW + w, seed2 pos2 + 2n + 64W + gW + w,
//                       seed3 pos3 + 8n + 64W + gW + w
//
// Kernels (every PRF block computed once):
//   k_gate_keystream  the 125 AND gates' zero-share words of every reference
//                     word the chunk touches: per (seed, gate) one contiguous
//                     stream segment -> HBM buffer G
//   k_reshare         own = z + F_p - F_{p-1}; writes reshared ml (u16) and
//                     diff0 = a*ml - b*hd (u32).  Two implementations: 504-lane
//                     tiles here (the tile's draws into shared memory one ChaCha
//                     block per thread per step, then thread = 4 lanes; the
//                     comparison-only path), lane-major in threshold_lm.cu
//                     (thread = 8 lanes, warp-cooperative windows; the batch
//                     query, where it runs beside the GEMM; see launch_threshold)
//   k_lift            bit-sliced (thread = 32 lanes): share_split of ml + the
//                     two adders {16,17} -> injected-bit rows
//   k_inject          bit_inject<15>, <16>, const-lifted into diff (tile /
//                     lane-major, as k_reshare)
//   k_msb             bit-sliced: share_split of diff + the 31-bit adder ->
//                     match-bit shares (the match words the OR tree of
//                     ortree.cu reads); DB-sharded queries: fused first
//                     bucketed MPC-OR level per warp instead
#include <cstdio>
#include <cstdlib>
#include <string>
#include <type_traits>

#include "common.cuh"
#include "kernels.h"

// min blocks per SM for the latency-bound bit-sliced kernels: 4 x 128 threads
// caps them at 128 registers (a few bytes of spill) for more resident warps;
// measured best of 1 / 4 / 5 / 6 (lift 11.9 -> 8.5 ms, msb 15.1 -> 13.2 ms
// per 10 serialized configs[1] queries)
#ifndef MSB_LB
#define MSB_LB 4
#endif
#ifndef LIFT_LB
#define LIFT_LB 4
#endif

namespace irisgpu {

namespace {

__device__ __forceinline__ void and3(const uint32_t x[3], const uint32_t y[3], const uint32_t f[3],
                                     uint32_t z[3]) {
#pragma unroll
  for (int p = 0; p < 3; ++p) {
    const int q = (p + 2) % 3;
    z[p] = (x[p] & y[p]) ^ (x[q] & y[p]) ^ (x[p] & y[q]) ^ f[p] ^ f[q];
  }
}

__device__ __forceinline__ uint64_t gate_base(const ThrArgs& A, int k, int g) {
  if ((uint32_t)g < A.nlift) return A.lift_base[k] + (uint64_t)g * A.W;
  return A.msb_base[k] + (uint64_t)(g - (int)A.nlift) * A.W;
}

}  // namespace

// ---------------------------------------------------------------- gate keystream
// Buffer G, per segment and (seed k, gate g) row kg: gate_row_words(nw) words,
// ChaCha block j of the row's reference range [E, E + nw) (E = gate_base + w_first)
// at word 8 j, i.e. word e at row + (e - E) + (E & 7).  Every block is a full,
// 64-byte-aligned 8-word store (padding words are never read): 16-byte vector
// stores instead of 8 strided u64 stores per thread (-32% on the ChaCha rate,
// measured).  block z -> segment, thread -> (seed k, gate g, block j)
__global__ void __launch_bounds__(256) k_gate_keystream(const __grid_constant__ ThrArgs A) {
  // grid: (blocks over one segment's (k, g, j) threads, 1, segment) -- no segment search
  const Seg& sg = A.segs[blockIdx.z];
  const uint64_t nw = (sg.lane_end - 1) / 64 - sg.w_first + 1;
  const uint32_t nb = (uint32_t)(nw / 8 + 2);  // blocks per (k, g) row
  const uint32_t local = blockIdx.x * blockDim.x + threadIdx.x;
  if (local >= 3u * A.ngates * nb) return;
  const uint32_t j = local % nb;
  const uint32_t kg = local / nb;
  const int k = kg / A.ngates, g = kg % A.ngates;
  const uint64_t E = gate_base(A, k, g) + sg.w_first;
  const uint64_t b = E / 8 + j;
  if (b > (E + nw - 1) / 8) return;
  uint32_t blk[16];
  chacha12_block(A.key[k], b, 0, blk);
  uint4* dst = reinterpret_cast<uint4*>(A.gate + sg.g_off + (uint64_t)kg * (8ull * nb) + 8ull * j);
#pragma unroll
  for (int q = 0; q < 4; ++q) dst[q] = make_uint4(blk[4 * q], blk[4 * q + 1], blk[4 * q + 2], blk[4 * q + 3]);
}

// ---------------------------------------------------------------- reshare
namespace {

// 4 lanes [L, L+4) of a dot array (u16 or u32) at src index i0 -> v[0..3]
// (`vec`: one aligned vector access; else per lane, lanes outside [lb, le) = 0)
template <typename T>
__device__ __forceinline__ void load4_at(const T* src, uint64_t i0, uint64_t L, uint64_t lb, uint64_t le, bool vec,
                                         uint32_t v[4]) {
  if (vec) {
    if (sizeof(T) == 2) {
      const uint2 x = *reinterpret_cast<const uint2*>(src + i0);
      v[0] = x.x & 0xFFFFu;
      v[1] = x.x >> 16;
      v[2] = x.y & 0xFFFFu;
      v[3] = x.y >> 16;
    } else {
      const uint4 x = *reinterpret_cast<const uint4*>(src + i0);
      v[0] = x.x;
      v[1] = x.y;
      v[2] = x.z;
      v[3] = x.w;
    }
    return;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) v[i] = (L + i >= lb && L + i < le) ? (uint32_t)src[i0 + i] : 0u;
}

// A field's dots of lanes [L, L+4): plain [col][row] planes (kstride 0), or (RP)
// the rotation pair's shared product P2 plus its own P1 / P3 (prep.cu)
template <typename T>
__device__ __forceinline__ void load4(const T* src, uint64_t kstride, const Seg& sg, uint64_t L, uint64_t lb,
                                      uint64_t le, bool vec, uint32_t v[4]) {
  if (!kstride) {
    load4_at<T>(src, sg.src + (L - sg.lane_begin), L, lb, le, vec, v);
    return;
  }
  const uint64_t i0 = sg.src_rp + (L - sg.lane_begin);
  uint32_t a[4];
  load4_at<T>(src, i0 + kstride, L, lb, le, vec, v);
  load4_at<T>(src, i0 + (sg.rp_sel == 1 ? 0 : 2 * kstride), L, lb, le, vec, a);
#pragma unroll
  for (int i = 0; i < 4; ++i) v[i] += a[i];
}

}  // namespace

// reshare_pair<KH, KM> (engine.cpp:80-106: hd lanes at stream offset 0, ml at
// n; zero_ring<K>, rep3.hpp:110-112: component k gains F(seed_k) and component
// k+1 loses it) followed by the comparison input:
//   mpc-lift   : ml_rs = ml (u16, lifted later), diff = a ml - b hd (partial)
//   const-lift : diff = a ml32 - const_lift(hd, b)      (engine.hpp:94-120)
//   no-lift    : diff = a ml32 - b hd32
//   plain-mask : diff = public_minus(ceil((1-2r) ml), hd) (engine.hpp:77-90)
//
// One CTA per kTile-lane tile of a segment (tiles start at the segment's first
// lane rounded down to a multiple of 4).  Phase 1: the tile's reshare draws -- per (dot, seed) the up to
// kTile/8 + 1 ChaCha12 blocks covering its kTile stream elements -- one block
// per thread per step at full occupancy (the k_gate_keystream pattern), the
// ring-width low bits of each element into shared memory.  Phase 2: thread = 4
// lanes, vector loads of the three parties' dots, own = z + F_k - F_{k-1},
// vector stores.  (The previous lane-major version held 6 blocks' windows per
// thread at 121 registers and 24% of the warps: 41% of the ChaCha rate.)
// The tile is kept small (6 KB of shared memory for 16-bit rings) so the CTAs
// fit beside the persistent GEMM's ~193 KB on the same SM: the threshold runs
// in the SMs' leftover resources while the GEMM streams.
// 504 lanes: any 504 consecutive stream elements lie in at most 64 ChaCha
// blocks, so phase 1 is 6 x 64 = 384 jobs = exactly 3 rounds of 128 threads
// (a 512-lane tile needs 65 blocks per window and a mostly idle 4th round)
constexpr int kTile = 504;
constexpr int kTileThreads = 128;

template <int V>
__global__ void __launch_bounds__(kTileThreads) k_reshare(const __grid_constant__ ThrArgs A) {
  using HT = typename std::conditional<V == kNoLift, uint32_t, uint16_t>::type;
  using MT = typename std::conditional<V == kConstLift || V == kNoLift, uint32_t, uint16_t>::type;
  constexpr uint32_t HM = V == kNoLift ? 0xFFFFFFFFu : 0xFFFFu;
  constexpr uint32_t MM = (V == kConstLift || V == kNoLift) ? 0xFFFFFFFFu : 0xFFFFu;
  constexpr int NDOT = V == kPlainMask ? 1 : 2;  // dot 0 = hd (offset 0), dot 1 = ml (offset n)
  constexpr int NB = (kTile + 6) / 8 + 1;          // blocks per (dot, seed) window
  using FH = HT;                                   // stored F words: the ring's width
  using FM = MT;
  __shared__ FH Fh[3][kTile];
  __shared__ FM Fm[NDOT - 1 ? 3 : 1][NDOT - 1 ? kTile : 1];
  const Seg& sg = A.segs[blockIdx.z];
  // tiles start at the segment's first lane rounded down to 4: a thread's 4 lanes never
  // straddle a 32-lane bit word (k_inject) nor a vector boundary
  const uint64_t T0 = (sg.lane_begin & ~3ull) + (uint64_t)blockIdx.x * kTile;
  if (T0 >= sg.lane_end) return;  // CTA-uniform
  const uint64_t lb = sg.lane_begin > T0 ? sg.lane_begin : T0;
  const uint64_t le = sg.lane_end < T0 + kTile ? sg.lane_end : T0 + kTile;
  const int lo = (int)(lb - T0), hi = (int)(le - T0);  // valid tile offsets [lo, hi)
  if (!A.no_reshare) {
    for (int j = threadIdx.x; j < NDOT * 3 * NB; j += blockDim.x) {
      const int d = j / (3 * NB), k = (j / NB) % 3, q = j % NB;
      const uint64_t e0 = A.pos[k] + (d ? A.n : 0) + T0;  // stream element of tile offset 0
      const uint64_t b = e0 / 8 + q;
      const int x0 = (int)(b * 8 - e0);  // tile offset of the block's word 0 (>= -7)
      if (x0 + 7 < lo || x0 >= hi) continue;
      uint32_t blk[16];
      chacha12_block(A.key[k], b, 0, blk);
#pragma unroll
      for (int w = 0; w < 8; ++w) {
        const int x = x0 + w;
        if (x < lo || x >= hi) continue;
        if (d == 0)
          Fh[k][x] = (FH)blk[2 * w];
        else
          Fm[k][x] = (FM)blk[2 * w];
      }
    }
    __syncthreads();
  }
  const uint64_t L = T0 + 4ull * threadIdx.x;
  if (L + 4 <= lb || L >= le) return;
  const bool full = L >= lb && L + 4 <= le;
  const int li = (int)(L - T0);
  const uint64_t src0 = sg.src + (L - sg.lane_begin);   // valid only when `full`
  const uint64_t hk = A.rp_kstride_h, mk = A.rp_kstride_m;
  const uint64_t rp0 = sg.src_rp + (L - sg.lane_begin);
  const uint64_t hs0 = hk ? rp0 : src0, ms0 = mk ? rp0 : src0;
  const HT* hd[3];
  const MT* ml[3];
  bool vin = full && !A.tap_rs_hd && hk % 4 == 0 && mk % 4 == 0;
  bool vout = full && !A.tap_rs_hd;
#pragma unroll
  for (int p = 0; p < 3; ++p) {
    hd[p] = static_cast<const HT*>(A.hd[p]);
    ml[p] = static_cast<const MT*>(A.ml[p]);
    vin = vin && ((reinterpret_cast<uintptr_t>(hd[p] + hs0) | reinterpret_cast<uintptr_t>(ml[p] + ms0)) &
                  (4 * sizeof(HT) - 1 | 4 * sizeof(MT) - 1)) == 0;
    vout = vout && (reinterpret_cast<uintptr_t>(A.diff + p * A.cstride + src0) & 15) == 0;
    if (V == kMpcLift) vout = vout && (reinterpret_cast<uintptr_t>(A.ml_rs + p * A.cstride + src0) & 7) == 0;
  }
  uint32_t d[3][4], m[3][4];
  if (V != kPlainMask) {
#pragma unroll
    for (int p = 0; p < 3; ++p) load4<MT>(ml[p], mk, sg, L, lb, le, vin, m[p]);
    if (!A.no_reshare) {
#pragma unroll
      for (int k = 0; k < 3; ++k)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const uint32_t f = Fm[k][li + i];
          m[k][i] += f;
          m[(k + 1) % 3][i] -= f;
        }
    }
#pragma unroll
    for (int p = 0; p < 3; ++p)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        m[p][i] &= MM;
        d[p][i] = A.a * m[p][i];
      }
    if (V == kMpcLift) {
#pragma unroll
      for (int p = 0; p < 3; ++p) {
        if (vout) {
          *reinterpret_cast<uint2*>(A.ml_rs + p * A.cstride + src0) =
              make_uint2(m[p][0] | (m[p][1] << 16), m[p][2] | (m[p][3] << 16));
        } else {
#pragma unroll
          for (int i = 0; i < 4; ++i)
            if (L + i >= lb && L + i < le)
              A.ml_rs[p * A.cstride + sg.src + (L + i - sg.lane_begin)] = (uint16_t)m[p][i];
        }
      }
    }
    if (A.tap_rs_ml) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if (L + i < lb || L + i >= le) continue;
#pragma unroll
        for (int p = 0; p < 3; ++p) {
          A.tap_rs_ml[p * A.n + L + i] = m[p][i];
          A.tap_ml32[p * A.n + L + i] = m[p][i];
        }
      }
    }
  }
  uint32_t (&h)[3][4] = m;  // reuse the registers
#pragma unroll
  for (int p = 0; p < 3; ++p) load4<HT>(hd[p], hk, sg, L, lb, le, vin, h[p]);
  if (!A.no_reshare) {
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint32_t f = Fh[k][li + i];
        h[k][i] += f;
        h[(k + 1) % 3][i] -= f;
      }
  }
#pragma unroll
  for (int p = 0; p < 3; ++p)
#pragma unroll
    for (int i = 0; i < 4; ++i) h[p][i] &= HM;
  if (V == kPlainMask) {
    // public popcount; diff = public_minus(t, hd): component 1 absorbs t (rep3.hpp:59-71)
    uint32_t cnt[4];
    load4<MT>(ml[0], mk, sg, L, lb, le, vin, cnt);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t t = (uint32_t)(int64_t)ceil(__dmul_rn(A.coef, (double)cnt[i]));
      d[0][i] = (t - h[0][i]) & 0xFFFFu;
      d[1][i] = (0u - h[1][i]) & 0xFFFFu;
      d[2][i] = (0u - h[2][i]) & 0xFFFFu;
    }
  } else {
#pragma unroll
    for (int p = 0; p < 3; ++p)
#pragma unroll
      for (int i = 0; i < 4; ++i) d[p][i] -= A.b * h[p][i];
  }
  if (vout) {
#pragma unroll
    for (int p = 0; p < 3; ++p)
      *reinterpret_cast<uint4*>(A.diff + p * A.cstride + src0) = make_uint4(d[p][0], d[p][1], d[p][2], d[p][3]);
    return;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if (L + i < lb || L + i >= le) continue;
    const uint64_t src = sg.src + (L + i - sg.lane_begin);
#pragma unroll
    for (int p = 0; p < 3; ++p) {
      A.diff[p * A.cstride + src] = d[p][i];
      if (A.tap_rs_hd) A.tap_rs_hd[p * A.n + L + i] = h[p][i];
    }
  }
}

// ---------------------------------------------------------------- bit-sliced circuits

namespace {

struct TaskCtx {
  Seg sg;
  uint64_t task, L0, vb, ve;
};

// blockIdx.z = segment, warp -> the segment's 1024-lane task (false: warp past the segment)
__device__ __forceinline__ bool task_ctx(const ThrArgs& A, TaskCtx& t) {
  t.sg = A.segs[blockIdx.z];
  const uint64_t nt = (t.sg.lane_end - 1) / 1024 - t.sg.lane_begin / 1024 + 1;
  const uint64_t tl = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (tl >= nt) return false;
  t.task = t.sg.task_begin + tl;
  t.L0 = (t.sg.q_first + tl) * 1024;
  t.vb = t.sg.lane_begin > t.L0 ? t.sg.lane_begin : t.L0;
  t.ve = t.sg.lane_end < t.L0 + 1024 ? t.sg.lane_end : t.L0 + 1024;
  return true;
}

// this thread's 32 lanes [Lt, Lt+32) as a valid-lane mask
__device__ __forceinline__ uint32_t valid_mask(const TaskCtx& t, uint64_t Lt) {
  if (!(t.ve > Lt && t.vb < Lt + 32)) return 0u;
  const uint32_t from = t.vb > Lt ? (uint32_t)(t.vb - Lt) : 0u;
  const uint32_t to = t.ve < Lt + 32 ? (uint32_t)(t.ve - Lt) : 32u;
  return (to >= 32 ? 0xFFFFFFFFu : ((1u << to) - 1)) & ~((1u << from) - 1);
}

// zero-share randomness of gate g for this thread's half reference word
__device__ __forceinline__ void gate_rand(const ThrArgs& A, const Seg& sg, uint64_t w64, int half, int g,
                                          uint32_t f[3]) {
  const uint64_t nwp = gate_row_words((sg.lane_end - 1) / 64 - sg.w_first + 1);
  const uint64_t* G = A.gate + sg.g_off + (w64 - sg.w_first);
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const uint32_t pad = (uint32_t)(gate_base(A, k, g) + sg.w_first) & 7u;  // k_gate_keystream layout
    f[k] = (uint32_t)(__ldg(G + (uint64_t)(k * A.ngates + g) * nwp + pad) >> (32 * half));
  }
}

// bit_extract_sum for one index M over summand rows R[c][j] (component c of
// summand c; rows j >= K are zero), evaluated position by position: chain
// gate t = j then full-adder gate j.  fa(j) = fa0 + j,
// ch(t) = min(ch0 + chs (t - 1), chmax).
template <int M, int K>
__device__ __forceinline__ void extract_bit(const ThrArgs& A, const Seg& sg, uint64_t w64, int half,
                                            const uint32_t (&R)[3][K], int fa0, int ch0, int chs, int chmax,
                                            uint32_t out[3]) {
  uint32_t carry[3] = {0, 0, 0}, chain[3] = {0, 0, 0};
  // gate randomness one step ahead: the loads of step j + 1 are in flight while
  // step j computes (the kernels are latency-bound on these L2 reads)
  uint32_t fc_next[3] = {0, 0, 0}, ff_next[3];
  gate_rand(A, sg, w64, half, fa0, ff_next);
#pragma unroll
  for (int j = 0; j < M; ++j) {
    uint32_t fc[3], ff[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      fc[c] = fc_next[c];
      ff[c] = ff_next[c];
    }
    if (j + 1 < M) {
      gate_rand(A, sg, w64, half, min(ch0 + chs * j, chmax), fc_next);  // chain gate of step j + 1
      gate_rand(A, sg, w64, half, fa0 + j + 1, ff_next);
    }
    uint32_t s[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) s[c] = j < K ? R[c][j] : 0u;
    if (j >= 1) {
      uint32_t u[3], v[3], res[3];
      if (j == 1) {
#pragma unroll
        for (int c = 0; c < 3; ++c) { u[c] = s[c]; v[c] = carry[c]; }
        and3(u, v, fc, res);
#pragma unroll
        for (int c = 0; c < 3; ++c) chain[c] = res[c];
      } else {
#pragma unroll
        for (int c = 0; c < 3; ++c) { u[c] = s[c] ^ chain[c]; v[c] = carry[c] ^ chain[c]; }
        and3(u, v, fc, res);
#pragma unroll
        for (int c = 0; c < 3; ++c) chain[c] ^= res[c];
      }
    }
    {
      uint32_t z[3];
      const uint32_t t1[3] = {s[0], 0u, s[2]};
      const uint32_t t2[3] = {0u, s[1], s[2]};
      and3(t1, t2, ff, z);
      carry[0] = z[0];
      carry[1] = z[1];
      carry[2] = z[2] ^ s[2];
    }
  }
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const uint32_t sM = M < K ? R[c][M < K ? M : 0] : 0u;
    out[c] = sM ^ carry[c] ^ (M >= 2 ? chain[c] : 0u);
  }
}

}  // namespace

// warp -> 1024-lane task, thread -> 32 lanes
__global__ void __launch_bounds__(128, LIFT_LB) k_lift(const __grid_constant__ ThrArgs A) {
  const int lane = threadIdx.x & 31;
  TaskCtx t;
  if (!task_ctx(A, t)) return;
  const uint64_t task = t.task;
  const uint64_t Lt = t.L0 + 32ull * lane;
  const uint32_t vm = valid_mask(t, Lt);
  if (vm == 0) return;  // lanes outside the segment: no gate randomness was generated for them
  uint32_t R[3][16];
#pragma unroll
  for (int p = 0; p < 3; ++p) {
    uint32_t a[32];
    const uint64_t so = t.sg.src + (Lt - t.sg.lane_begin);
    if (vm == 0xFFFFFFFFu && (reinterpret_cast<uintptr_t>(A.ml_rs + p * A.cstride + so) & 15) == 0) {
      const uint4* src = reinterpret_cast<const uint4*>(A.ml_rs + p * A.cstride + so);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint4 x = src[q];
        const uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          a[8 * q + 2 * i] = w[i] & 0xFFFFu;
          a[8 * q + 2 * i + 1] = w[i] >> 16;
        }
      }
    } else if (vm == 0xFFFFFFFFu) {
      const uint16_t* src = A.ml_rs + p * A.cstride + so;
#pragma unroll
      for (int i = 0; i < 32; ++i) a[i] = src[i];
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i)
        a[i] = ((vm >> i) & 1) ? A.ml_rs[p * A.cstride + t.sg.src + (Lt + i - t.sg.lane_begin)] : 0u;
    }
    transpose32(a);
#pragma unroll
    for (int j = 0; j < 16; ++j) R[p][j] = a[j];
  }
  const uint64_t w64 = Lt / 64;
  const int half = lane & 1;
  uint32_t b16[3], b17[3];
  extract_bit<16, 16>(A, t.sg, w64, half, R, 0, 33, 2, 63, b16);
  extract_bit<17, 16>(A, t.sg, w64, half, R, 16, 34, 2, 63, b17);
  const uint64_t o = task * 32 + lane;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    A.bits[c * A.nbits + o] = b16[c];
    A.bits[(3 + c) * A.nbits + o] = b17[c];
  }
}

// bit_inject<15>(bit17) then bit_inject<16>(bit16) (convert.hpp:84-155), three
// parties at once: P1's c1 (seed 1, one draw per lane) and P3's c3 (seed 3,
// (c3, w0, w1) per lane, only c3 enters the sharing) give b1 = c1, b3 = c3,
// b2 = x - b1 - b3 (mod 2^W), each injected bit lifted by 2^17 / 2^16 and
// subtracted, times a, from diff.  One CTA per kTile-lane tile: phase 1 computes
// the tile's 2 x (kTile/8 + 1 + 3 kTile/8 + 1) ChaCha12 blocks one per thread
// per step into shared memory (c1, c3 low halves; 4 KB), phase 2 applies them,
// thread = 4 lanes.
__global__ void __launch_bounds__(kTileThreads) k_inject(const __grid_constant__ ThrArgs A) {
  __shared__ uint16_t C[2][2][kTile];  // [inject 15 / 16][c1 / c3][lane]
  const Seg& sg = A.segs[blockIdx.z];
  // tiles start at the segment's first lane rounded down to 4: a thread's 4 lanes never
  // straddle a 32-lane bit word (k_inject) nor a vector boundary
  const uint64_t T0 = (sg.lane_begin & ~3ull) + (uint64_t)blockIdx.x * kTile;
  if (T0 >= sg.lane_end) return;  // CTA-uniform
  const uint64_t lb = sg.lane_begin > T0 ? sg.lane_begin : T0;
  const uint64_t le = sg.lane_end < T0 + kTile ? sg.lane_end : T0 + kTile;
  const int lo = (int)(lb - T0), hi = (int)(le - T0);
  const uint64_t n = A.n;
  constexpr int J1 = (kTile + 6) / 8 + 1, J3 = (3 * kTile + 6) / 8 + 1, JW = J1 + J3;
  for (int j = threadIdx.x; j < 2 * JW; j += blockDim.x) {
    const int which = j / JW, q = j % JW;
    const bool s3 = q >= J1;
    // stream element of tile offset 0: seed 1 at inj_base + (n for inject16) + T0,
    // seed 3 at inj_base + (3n for inject16) + 3 T0 (element 3x of lane x is c3)
    const uint64_t e0 = s3 ? A.inj_base[2] + (which ? 3 * n : 0) + 3 * T0 : A.inj_base[0] + (which ? n : 0) + T0;
    const uint64_t b = e0 / 8 + (s3 ? q - J1 : q);
    const int x0 = (int)(b * 8 - e0);  // element offset of the block's word 0 (>= -7)
    if (s3 ? (x0 + 7 < 3 * lo || x0 > 3 * (hi - 1)) : (x0 + 7 < lo || x0 >= hi)) continue;
    uint32_t blk[16];
    chacha12_block(A.key[s3 ? 2 : 0], b, 0, blk);
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      const int x = x0 + w;
      if (!s3) {
        if (x >= lo && x < hi) C[which][0][x] = (uint16_t)blk[2 * w];
      } else if (x >= 0 && x % 3 == 0 && x / 3 >= lo && x / 3 < hi) {
        C[which][1][x / 3] = (uint16_t)blk[2 * w];
      }
    }
  }
  __syncthreads();
  const uint64_t L = T0 + 4ull * threadIdx.x;
  if (L + 4 <= lb || L >= le) return;
  const int li = (int)(L - T0);
  // injected bits: the k_lift thread that owns these lanes (its 1024-lane task, lane word)
  const uint64_t task = sg.task_begin + (L / 1024 - sg.q_first);
  const uint64_t o = task * 32 + (L % 1024) / 32;
  const int sh = (int)(L % 32);
  const uint32_t x17 = (A.bits[3 * A.nbits + o] ^ A.bits[4 * A.nbits + o] ^ A.bits[5 * A.nbits + o]) >> sh;
  const uint32_t x16 = (A.bits[0 * A.nbits + o] ^ A.bits[1 * A.nbits + o] ^ A.bits[2 * A.nbits + o]) >> sh;
  uint32_t d[3][4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    d[0][i] = d[1][i] = d[2][i] = 0u;
#pragma unroll
    for (int which = 0; which < 2; ++which) {
      const uint32_t x = which == 0 ? x17 : x16;
      const uint32_t mask = which == 0 ? 0x7FFFu : 0xFFFFu;
      const int shift = which == 0 ? 17 : 16;
      const uint32_t b1 = C[which][0][li + i] & mask;
      const uint32_t b3 = C[which][1][li + i] & mask;
      const uint32_t b2 = (((x >> i) & 1u) - b1 - b3) & mask;
      d[0][i] += b1 << shift;
      d[1][i] += b2 << shift;
      d[2][i] += b3 << shift;
    }
  }
  const uint64_t src0 = sg.src + (L - sg.lane_begin);
  bool vec = L >= lb && L + 4 <= le && !A.tap_ml32;
#pragma unroll
  for (int p = 0; p < 3; ++p) vec = vec && (reinterpret_cast<uintptr_t>(A.diff + p * A.cstride + src0) & 15) == 0;
  if (vec) {
#pragma unroll
    for (int p = 0; p < 3; ++p) {
      uint4* dd = reinterpret_cast<uint4*>(A.diff + p * A.cstride + src0);
      uint4 x = *dd;
      x.x -= A.a * d[p][0];
      x.y -= A.a * d[p][1];
      x.z -= A.a * d[p][2];
      x.w -= A.a * d[p][3];
      *dd = x;
    }
    return;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint64_t ln = L + i;
    if (ln < lb || ln >= le) continue;
    const uint64_t src = sg.src + (ln - sg.lane_begin);
#pragma unroll
    for (int p = 0; p < 3; ++p) {
      A.diff[p * A.cstride + src] -= A.a * d[p][i];
      if (A.tap_ml32) A.tap_ml32[p * n + ln] -= d[p][i];
    }
  }
}

namespace {

__device__ __noinline__ void fused_or(const ThrArgs& A, const Seg& sg, uint64_t task, const uint32_t bit_in[3],
                                      int lane, uint64_t (*orr)[40]) {
  // 36 AND gates per warp, randomness from the query's fused-OR stream (elements E0 + gate)
  const uint64_t E0 = A.or_elem_base + task * 64;
  __syncwarp();
  if (lane < 18) {
    const int k = lane / 6, bo = lane % 6;
    const uint64_t b = E0 / 8 + bo;
    if (b <= (E0 + 35) / 8) {
      uint32_t blk[16];
      chacha12_block(A.key[k], b, A.or_stream, blk);
#pragma unroll
      for (int w = 0; w < 8; ++w) {
        const uint64_t e = b * 8 + w;
        if (e >= E0 && e < E0 + 36) orr[k][e - E0] = chacha_word(blk, w);
      }
    }
  }
  __syncwarp();
  uint32_t x[3] = {bit_in[0], bit_in[1], bit_in[2]};
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    uint32_t y[3], f[3], z[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) y[c] = __shfl_down_sync(0xffffffffu, x[c], o);
    const int gid = min(32 - 2 * o + lane, 30);
#pragma unroll
    for (int k = 0; k < 3; ++k) f[k] = (uint32_t)orr[k][gid];
    and3(x, y, f, z);
#pragma unroll
    for (int c = 0; c < 3; ++c) x[c] = x[c] ^ y[c] ^ z[c];
  }
  if (lane == 0) {
    int lvl = 0;
#pragma unroll
    for (int h = 16; h >= 1; h >>= 1, ++lvl) {
      const uint32_t m = (1u << h) - 1;
      uint32_t lo_[3], hi_[3], f[3], z[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) { lo_[c] = x[c] & m; hi_[c] = (x[c] >> h) & m; }
#pragma unroll
      for (int k = 0; k < 3; ++k) f[k] = (uint32_t)orr[k][31 + lvl] & m;
      and3(lo_, hi_, f, z);
#pragma unroll
      for (int c = 0; c < 3; ++c) x[c] = lo_[c] ^ hi_[c] ^ (z[c] & m);
    }
    const uint64_t slot = (uint64_t)sg.slot + (task - sg.task_begin);
#pragma unroll
    for (int c = 0; c < 3; ++c) A.partial[c * A.nslots + slot] = (uint8_t)(x[c] & 1u);
  }
}

}  // namespace

// warp -> 1024-lane task: msb<KC> of diff (circuits.hpp:300-306), outputs,
// fused first OR level.  Gates: FA j -> nlift + j, chain t -> nlift + KC - 1 + (t - 1).
template <int KC>
__global__ void __launch_bounds__(128, MSB_LB) k_msb(const __grid_constant__ ThrArgs A) {
  const int lane = threadIdx.x & 31;
  TaskCtx t;
  if (!task_ctx(A, t)) return;
  const uint64_t task = t.task;
  const uint64_t Lt = t.L0 + 32ull * lane;
  const uint32_t vm = valid_mask(t, Lt);
  uint32_t D[3][32];
#pragma unroll
  for (int p = 0; p < 3; ++p) {
    const uint64_t so = t.sg.src + (Lt - t.sg.lane_begin);
    if (vm == 0xFFFFFFFFu && (reinterpret_cast<uintptr_t>(A.diff + p * A.cstride + so) & 15) == 0) {
      const uint4* src = reinterpret_cast<const uint4*>(A.diff + p * A.cstride + so);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const uint4 x = src[q];
        D[p][4 * q] = x.x;
        D[p][4 * q + 1] = x.y;
        D[p][4 * q + 2] = x.z;
        D[p][4 * q + 3] = x.w;
      }
    } else if (vm == 0xFFFFFFFFu) {
      const uint32_t* src = A.diff + p * A.cstride + so;
#pragma unroll
      for (int i = 0; i < 32; ++i) D[p][i] = src[i];
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i)
        D[p][i] = ((vm >> i) & 1) ? A.diff[p * A.cstride + t.sg.src + (Lt + i - t.sg.lane_begin)] : 0u;
    }
    if (A.tap_diff) {
      for (int i = 0; i < 32; ++i)
        if ((vm >> i) & 1) A.tap_diff[p * A.n + Lt + i] = D[p][i];
    }
    transpose32(D[p]);
  }
  uint32_t bit[3] = {0u, 0u, 0u};
  // rows >= KC of the transposed diff are never read (extract_bit<KC - 1, 32> touches rows <= KC - 1)
  const int nl = (int)A.nlift;
  if (vm) extract_bit<KC - 1, 32>(A, t.sg, Lt / 64, lane & 1, D, nl, nl + KC - 1, 1, nl + 2 * KC - 4, bit);
#pragma unroll
  for (int c = 0; c < 3; ++c) bit[c] &= vm;
  if (A.tap_msb) {
    for (int i = 0; i < 32; ++i)
      if ((vm >> i) & 1)
        for (int c = 0; c < 3; ++c) A.tap_msb[c * A.n + Lt + i] = (bit[c] >> i) & 1;
  }
  if (A.match[0] && vm) {
    const uint64_t wi = Lt / 32 - A.match_w0;
#pragma unroll
    for (int c = 0; c < 3; ++c) atomicOr(&A.match[c][wi], bit[c]);
  }
  __shared__ uint64_t orr[4][3][40];
  if (t.sg.slot >= 0) fused_or(A, t.sg, task, bit, lane, orr[threadIdx.x >> 5]);
}

// ---------------------------------------------------------------- comparison phase alone

// party_comparison_only's parse_rep_shares (src/engine.cpp:455-467): lane i of
// party p's payload is (own, prev) as two little-endian ring elements of
// `width` bytes; component p = own_p, and prev_p must equal own_{p-1} (the
// replication cross-check of a RepShare).  width 8 = the plain-mask public ml
// (one LE u64 per lane, identical at every party; out has one plane).
__global__ void k_parse_lane_shares(const uint8_t* __restrict__ p1, const uint8_t* __restrict__ p2,
                                    const uint8_t* __restrict__ p3, uint64_t lanes, int width, void* out,
                                    int* bad) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= lanes) return;
  const uint8_t* P[3] = {p1, p2, p3};
  auto rd = [&](const uint8_t* p, uint64_t off, int w) {
    uint64_t v = 0;
    for (int b = 0; b < w; ++b) v |= (uint64_t)p[off + b] << (8 * b);
    return v;
  };
  if (width == 8) {
    const uint64_t a = rd(P[0], 8 * i, 8), b = rd(P[1], 8 * i, 8), c = rd(P[2], 8 * i, 8);
    if (a != b || a != c) atomicOr(bad, 1);
    static_cast<uint16_t*>(out)[i] = (uint16_t)a;
    return;
  }
  uint64_t own[3], prev[3];
  for (int p = 0; p < 3; ++p) {
    own[p] = rd(P[p], 2ull * width * i, width);
    prev[p] = rd(P[p], 2ull * width * i + width, width);
  }
  for (int p = 0; p < 3; ++p) {
    if (prev[p] != own[(p + 2) % 3]) atomicOr(bad, 1);
    if (width == 2)
      static_cast<uint16_t*>(out)[p * lanes + i] = (uint16_t)own[p];
    else
      static_cast<uint32_t*>(out)[p * lanes + i] = (uint32_t)own[p];
  }
}

void launch_parse_lane_shares(const uint8_t* const p[3], uint64_t lanes, int width, void* out, int* bad,
                              cudaStream_t st) {
  if (!lanes) return;
  k_parse_lane_shares<<<(unsigned)((lanes + 255) / 256), 256, 0, st>>>(p[0], p[1], p[2], lanes, width, out, bad);
}

// party_or_tree_only's payload (engine.cpp:517-532): per 64-lane word
// (own u64, prev u64) of party p -> component words [3][2 * words] (u32 halves)
__global__ void k_parse_bit_shares(const uint8_t* __restrict__ p1, const uint8_t* __restrict__ p2,
                                   const uint8_t* __restrict__ p3, uint64_t words, uint64_t lanes,
                                   uint32_t* __restrict__ out, int* bad) {
  const uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (w >= words) return;
  const uint8_t* P[3] = {p1, p2, p3};
  uint64_t own[3], prev[3];
  for (int p = 0; p < 3; ++p) {
    own[p] = prev[p] = 0;
    for (int b = 0; b < 8; ++b) {
      own[p] |= (uint64_t)P[p][16 * w + b] << (8 * b);
      prev[p] |= (uint64_t)P[p][16 * w + 8 + b] << (8 * b);
    }
  }
  const uint64_t valid = (lanes - 64 * w) >= 64 ? ~0ull : ((1ull << (lanes - 64 * w)) - 1);
  for (int p = 0; p < 3; ++p) {
    if (prev[p] != own[(p + 2) % 3]) atomicOr(bad, 1);
    out[p * 2 * words + 2 * w] = (uint32_t)(own[p] & valid);
    out[p * 2 * words + 2 * w + 1] = (uint32_t)((own[p] & valid) >> 32);
  }
}

void launch_parse_bit_shares(const uint8_t* const p[3], uint64_t words, uint64_t lanes, uint32_t* out, int* bad,
                             cudaStream_t st) {
  if (!words) return;
  k_parse_bit_shares<<<(unsigned)((words + 255) / 256), 256, 0, st>>>(p[0], p[1], p[2], words, lanes, out, bad);
}

template <typename T>
__global__ void k_rp_tap(const T* __restrict__ P, uint32_t nparty, uint64_t ncols, uint32_t rot, uint64_t nr,
                         uint64_t kstride, T* __restrict__ out, uint64_t n, uint64_t S, uint64_t row0) {
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (tid >= nparty * ncols * nr) return;
  const uint64_t row = tid % nr, pc = tid / nr, col = pc % ncols, p = pc / ncols;
  const uint32_t npr = (rot + 1) / 2, j = (uint32_t)(col % rot);
  const uint64_t cp = (col / rot) * npr + j / 2;
  const uint64_t i = p * (npr * (ncols / rot)) * nr + cp * nr + row;  // party p's P1 plane
  out[p * n + col * S + row0 + row] = (T)(P[i + kstride] + P[i + ((j & 1) ? 0 : 2 * kstride)]);
}

void launch_rp_tap(const void* P, int elem_bytes, uint32_t nparty, uint64_t ncols, uint32_t rot, uint64_t nr,
                   uint64_t kstride, void* out, uint64_t n, uint64_t S, uint64_t row0, cudaStream_t st) {
  const uint64_t tot = nparty * ncols * nr;
  const unsigned g = (unsigned)((tot + 255) / 256);
  if (elem_bytes == 2)
    k_rp_tap<uint16_t><<<g, 256, 0, st>>>(static_cast<const uint16_t*>(P), nparty, ncols, rot, nr, kstride,
                                           static_cast<uint16_t*>(out), n, S, row0);
  else
    k_rp_tap<uint32_t><<<g, 256, 0, st>>>(static_cast<const uint32_t*>(P), nparty, ncols, rot, nr, kstride,
                                           static_cast<uint32_t*>(out), n, S, row0);
}

// Row-sampled L1 tap: for every sampled DB row inside this chunk, the per-party
// dots of all its columns -> out[p * out_pstride + col * k + i] (i = the row's
// index in the sample).  Plain [party][col][row] dots, or RP planes (kstride > 0).
template <typename T>
__global__ void k_tap_rows(const T* __restrict__ P, uint32_t nparty, uint64_t ncols, uint32_t rot, uint64_t nr,
                           uint64_t kstride, const uint64_t* __restrict__ rows, uint32_t k, uint64_t row0,
                           T* __restrict__ out, uint64_t out_pstride) {
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (tid >= (uint64_t)nparty * ncols * k) return;
  const uint32_t i = (uint32_t)(tid % k);
  const uint64_t pc = tid / k, col = pc % ncols, p = pc / ncols;
  const uint64_t row = rows[i];
  if (row < row0 || row >= row0 + nr) return;
  const uint64_t rr = row - row0;
  T v;
  if (kstride == 0) {
    v = P[(p * ncols + col) * nr + rr];
  } else {
    const uint32_t npr = (rot + 1) / 2, j = (uint32_t)(col % rot);
    const uint64_t cp = (col / rot) * npr + j / 2;
    const uint64_t x = p * (npr * (ncols / rot)) * nr + cp * nr + rr;
    v = (T)(P[x + kstride] + P[x + ((j & 1) ? 0 : 2 * kstride)]);
  }
  out[p * out_pstride + col * k + i] = v;
}

void launch_tap_rows(const void* P, int elem_bytes, uint32_t nparty, uint64_t ncols, uint32_t rot, uint64_t nr,
                     uint64_t kstride, const uint64_t* rows, uint32_t k, uint64_t row0, void* out,
                     uint64_t out_pstride, cudaStream_t st) {
  const uint64_t tot = (uint64_t)nparty * ncols * k;
  if (!tot) return;
  const unsigned g = (unsigned)((tot + 255) / 256);
  if (elem_bytes == 2)
    k_tap_rows<uint16_t><<<g, 256, 0, st>>>(static_cast<const uint16_t*>(P), nparty, ncols, rot, nr, kstride, rows, k,
                                            row0, static_cast<uint16_t*>(out), out_pstride);
  else
    k_tap_rows<uint32_t><<<g, 256, 0, st>>>(static_cast<const uint32_t*>(P), nparty, ncols, rot, nr, kstride, rows, k,
                                            row0, static_cast<uint32_t*>(out), out_pstride);
}

void launch_threshold(const ThrArgs& a, cudaStream_t st) {
  launch_threshold_front(a, st);
  launch_threshold_back(a, st);
}

// front half: the gate keystream and the reshare (the only readers of the dot
// outputs); back half: lift, inject, msb (the latency-bound bit-sliced adders)
void launch_threshold_front(const ThrArgs& a, cudaStream_t st) { launch_threshold_part(a, st, 1); }
void launch_threshold_back(const ThrArgs& a, cudaStream_t st) { launch_threshold_part(a, st, 2); }

void launch_threshold_part(const ThrArgs& a, cudaStream_t st, int parts) {
  if (!a.ntasks) return;
  // leave-one-out timing hook (results are WRONG with it, so it also needs
  // IRISMPC_TIMING_ONLY=1): IRISMPC_SKIP_KERNELS=keystream,reshare,lift,inject,msb
  static const std::string skip = [] {
    const char* e = std::getenv("IRISMPC_SKIP_KERNELS");
    const char* ok = std::getenv("IRISMPC_TIMING_ONLY");
    if (e && !(ok && ok[0] == '1')) {
      std::fprintf(stderr, "irismpc: IRISMPC_SKIP_KERNELS ignored (set IRISMPC_TIMING_ONLY=1 to accept wrong results)\n");
      return std::string();
    }
    return e ? std::string(",") + e + "," : std::string();
  }();
  auto on = [&](const char* k) { return skip.empty() || skip.find(std::string(",") + k + ",") == std::string::npos; };
  // reshare / inject: one CTA per kTile-lane tile of a segment
  const dim3 tile_blocks((unsigned)((a.task_seg_max * 1024ull + 3 + kTile - 1) / kTile), 1, a.nsegs);
  const dim3 task_blocks((a.task_seg_max + 3) / 4, 1, a.nsegs);  // 4 warps (tasks) per 128-thread block
  // Which reshare / inject kernels: the tile kernels run 1.5x (reshare) faster
  // standalone (comparison-only path, serial profile), but beside the persistent
  // GEMM of a batch query the lane-major kernels keep the threshold stream
  // shorter (configs[2]: 432-437 vs 483 ms per query, same box, A/B in
  // profiles/r2_threshold_ab.md), so the batch query uses those.
  // IRISMPC_THR_KERNELS=tile|lm overrides (A/B hook).
  static const int force = [] {
    const char* e = std::getenv("IRISMPC_THR_KERNELS");
    return !e ? -1 : (std::string(e) == "tile" ? 1 : 0);
  }();
  const bool lm = force >= 0 ? force == 0 : !a.tile_kernels;
  if (parts & 1) {
    void* h = prof_begin(st);
    if (on("keystream")) k_gate_keystream<<<dim3((a.ks_seg_threads + 255) / 256, 1, a.nsegs), 256, 0, st>>>(a);
    prof_end(h, "k_gate_keystream", st);
    debug_check("k_gate_keystream", st);
    h = prof_begin(st);
    if (!on("reshare")) {
    } else if (lm) {
      launch_reshare_lm(a, st);
    } else {
      switch (a.variant) {
        case kPlainMask: k_reshare<kPlainMask><<<tile_blocks, kTileThreads, 0, st>>>(a); break;
        case kMpcLift: k_reshare<kMpcLift><<<tile_blocks, kTileThreads, 0, st>>>(a); break;
        case kConstLift: k_reshare<kConstLift><<<tile_blocks, kTileThreads, 0, st>>>(a); break;
        default: k_reshare<kNoLift><<<tile_blocks, kTileThreads, 0, st>>>(a); break;
      }
    }
    prof_end(h, "k_reshare", st);
    debug_check("k_reshare", st);
  }
  if (!(parts & 2)) return;
  if (a.variant == kMpcLift) {
    void* h = prof_begin(st);
    if (on("lift")) k_lift<<<task_blocks, 128, 0, st>>>(a);
    prof_end(h, "k_lift", st);
    debug_check("k_lift", st);
    h = prof_begin(st);
    if (!on("inject")) {
    } else if (lm) {
      launch_inject_lm(a, st);
    } else {
      k_inject<<<tile_blocks, kTileThreads, 0, st>>>(a);
    }
    prof_end(h, "k_inject", st);
    debug_check("k_inject", st);
  }
  void* h = prof_begin(st);
  if (!on("msb")) {
  } else if (a.variant == kPlainMask) {
    k_msb<16><<<task_blocks, 128, 0, st>>>(a);
  } else {
    k_msb<32><<<task_blocks, 128, 0, st>>>(a);
  }
  prof_end(h, "k_msb", st);
  debug_check("k_msb", st);
}

}  // namespace irisgpu
