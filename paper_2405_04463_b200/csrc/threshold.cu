// K4: the mpc-lift threshold comparison for all three parties of a lane tile.
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
//   inject<16>: seed1 -> pos1 + 3n + 64W + i,    seed3 -> pos3 + 5n + 64W + 3i
//   msb gate g (0..60): seed1 pos1 + 4n + 64W + gW + w, seed2 pos2 + 2n + 64W + gW + w,
//                       seed3 pos3 + 8n + 64W + gW + w
//
// Work unit: one warp = 1024 consecutive global lanes (16 reference words);
// one thread = 32 lanes, bit-sliced in u32 registers.  PRF blocks are produced
// warp-cooperatively (each thread computes whole ChaCha12 blocks) and handed
// over through shared memory.  Finally the warp ORs its valid lanes (all in
// one person group) with MPC OR gates into one shared bit (the first level of
// the bucketed OR reduction; randomness from stream id 1).
#include "common.cuh"
#include "kernels.h"

namespace irisgpu {

namespace {

constexpr int kWarps = 4;
constexpr int kGateWin = 5;  // steps staged per refill (<= 10 gates)

struct WarpSmem {
  uint32_t w32[3][1024];
  uint16_t s16[4][1024];
  uint64_t gr[2 * kGateWin][3][16];
};

__device__ __forceinline__ void and3(const uint32_t x[3], const uint32_t y[3], const uint32_t f[3],
                                     uint32_t z[3]) {
#pragma unroll
  for (int p = 0; p < 3; ++p) {
    const int q = (p + 2) % 3;
    z[p] = (x[p] & y[p]) ^ (x[q] & y[p]) ^ (x[p] & y[q]) ^ f[p] ^ f[q];
  }
}

// dst[i] = low 16 bits of stream element first + i*step, i < count.
__device__ __forceinline__ void warp_fill16(const SeedKey& key, uint64_t first, uint32_t count,
                                            uint32_t step, uint16_t* dst, int lane) {
  const uint64_t last = first + (uint64_t)(count - 1) * step;
  const uint64_t b_lo = first / 8, b_hi = last / 8;
  for (uint64_t b = b_lo + lane; b <= b_hi; b += 32) {
    uint32_t blk[16];
    chacha12_block(key, b, 0, blk);
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      const uint64_t e = b * 8 + w;
      if (e >= first && e <= last) {
        const uint32_t d = (uint32_t)(e - first);
        if (step == 1) {
          dst[d] = (uint16_t)blk[2 * w];
        } else if (d % step == 0) {
          dst[d / step] = (uint16_t)blk[2 * w];
        }
      }
    }
  }
  __syncwarp();
}

// Stage the 16 words (w0 .. w0+15) of `ng` gates for all three seeds.
__device__ __forceinline__ void stage_gates(WarpSmem& sm, const ThrArgs& A, const uint64_t base[3],
                                            const int* gid, int ng, uint64_t w0, int lane) {
  __syncwarp();
  for (int s = lane; s < ng * 9; s += 32) {
    const int gi = s / 9, k = (s % 9) / 3, bo = s % 3;
    if (gid[gi] < 0) continue;
    const uint64_t e0 = base[k] + (uint64_t)gid[gi] * A.W + w0;
    const uint64_t b = e0 / 8 + bo;
    if (b > (e0 + 15) / 8) continue;
    uint32_t blk[16];
    chacha12_block(A.key[k], b, 0, blk);
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      const uint64_t e = b * 8 + w;
      if (e >= e0 && e < e0 + 16) sm.gr[gi][k][e - e0] = chacha_word(blk, w);
    }
  }
  __syncwarp();
}

__device__ __forceinline__ void gate_rand(const WarpSmem& sm, int gi, int lane, uint32_t f[3]) {
#pragma unroll
  for (int k = 0; k < 3; ++k) f[k] = (uint32_t)(sm.gr[gi][k][lane >> 1] >> (32 * (lane & 1)));
}

// bit_extract_sum for one index M over summand bit rows R[c][j] (component c
// of summand c; rows j >= K are zero), evaluated position by position: at step
// j the ripple-chain gate t = j (if any) then the full-adder gate j.  Gate ids:
// fa(j) = fa0 + j; ch(t) = min(ch0 + chs * (t - 1), chmax).
template <int M, int K>
__device__ __forceinline__ void extract_bit(WarpSmem& sm, const ThrArgs& A, const uint64_t base[3],
                                            uint64_t w0, int lane, const uint32_t (&R)[3][K],
                                            int fa0, int ch0, int chs, int chmax, uint32_t out[3]) {
  uint32_t carry[3] = {0, 0, 0}, chain[3] = {0, 0, 0};
#pragma unroll
  for (int j = 0; j < M; ++j) {
    if (j % kGateWin == 0) {
      int gid[2 * kGateWin];
#pragma unroll
      for (int i = 0; i < kGateWin; ++i) {
        const int jj = j + i;
        gid[i] = jj < M ? fa0 + jj : -1;
        gid[kGateWin + i] = (jj >= 1 && jj <= M - 1) ? min(ch0 + chs * (jj - 1), chmax) : -1;
      }
      stage_gates(sm, A, base, gid, 2 * kGateWin, w0, lane);
    }
    uint32_t s[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) s[c] = j < K ? R[c][j] : 0u;
    if (j >= 1) {
      uint32_t f[3], u[3], v[3], res[3];
      gate_rand(sm, kGateWin + (j % kGateWin), lane, f);
      if (j == 1) {
#pragma unroll
        for (int c = 0; c < 3; ++c) { u[c] = s[c]; v[c] = carry[c]; }
        and3(u, v, f, res);
#pragma unroll
        for (int c = 0; c < 3; ++c) chain[c] = res[c];
      } else {
#pragma unroll
        for (int c = 0; c < 3; ++c) { u[c] = s[c] ^ chain[c]; v[c] = carry[c] ^ chain[c]; }
        and3(u, v, f, res);
#pragma unroll
        for (int c = 0; c < 3; ++c) chain[c] ^= res[c];
      }
    }
    {
      uint32_t f[3], z[3];
      gate_rand(sm, j % kGateWin, lane, f);
      const uint32_t t1[3] = {s[0], 0u, s[2]};
      const uint32_t t2[3] = {0u, s[1], s[2]};
      and3(t1, t2, f, z);
      carry[0] = z[0];
      carry[1] = z[1];
      carry[2] = z[2] ^ s[2];
    }
  }
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const uint32_t sm_ = M < K ? R[c][M < K ? M : 0] : 0u;
    out[c] = sm_ ^ carry[c] ^ (M >= 2 ? chain[c] : 0u);
  }
}

}  // namespace

__global__ void __launch_bounds__(kWarps * 32) k_threshold(const ThrArgs A) {
  extern __shared__ uint8_t smem_raw[];
  WarpSmem* all = reinterpret_cast<WarpSmem*>(smem_raw);
  const int wib = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  WarpSmem& sm = all[wib];
  const uint64_t task = (uint64_t)blockIdx.x * kWarps + wib;
  if (task >= A.ntasks) return;

  // segment of this task (warp-uniform binary search)
  uint32_t lo = 0, hi = A.nsegs - 1;
  while (lo < hi) {
    const uint32_t mid = (lo + hi + 1) >> 1;
    if (A.segs[mid].task_begin <= task) lo = mid; else hi = mid - 1;
  }
  const Seg sg = A.segs[lo];
  const uint64_t q = sg.q_first + (task - sg.task_begin);
  const uint64_t L0 = q * 1024;
  const uint64_t vb = sg.lane_begin > L0 ? sg.lane_begin : L0;
  const uint64_t ve = sg.lane_end < L0 + 1024 ? sg.lane_end : L0 + 1024;
  const uint64_t n = A.n, W = A.W;
  const uint64_t w0 = L0 / 64;  // first reference word of the warp (16 per warp)

  // ---- load additive dot shares (coalesced) --------------------------------
  for (int e = lane; e < 1024; e += 32) {
    const uint64_t ln = L0 + e;
    const bool ok = ln >= vb && ln < ve;
    const uint64_t src = sg.src + (ln - sg.lane_begin);
#pragma unroll
    for (int p = 0; p < 3; ++p) {
      sm.w32[p][e] = ok ? A.ml[p][src] : 0u;
      sm.s16[p][e] = ok ? A.hd[p][src] : (uint16_t)0;
    }
  }
  __syncwarp();

  // ---- reshare_pair: own_p = z_p + F(seed_p) - F(seed_{p-1}) ---------------
  for (int k = 0; k < 3; ++k) {
    warp_fill16(A.key[k], A.pos[k] + n + L0, 1024, 1, sm.s16[3], lane);
#pragma unroll 4
    for (int i = 0; i < 32; ++i) {
      const int e = lane * 32 + i;
      const uint32_t f = sm.s16[3][e];
      sm.w32[k][e] += f;
      sm.w32[(k + 1) % 3][e] -= f;
    }
    __syncwarp();
    warp_fill16(A.key[k], A.pos[k] + L0, 1024, 1, sm.s16[3], lane);
#pragma unroll 4
    for (int i = 0; i < 32; ++i) {
      const int e = lane * 32 + i;
      const uint16_t f = sm.s16[3][e];
      sm.s16[k][e] = (uint16_t)(sm.s16[k][e] + f);
      sm.s16[(k + 1) % 3][e] = (uint16_t)(sm.s16[(k + 1) % 3][e] - f);
    }
    __syncwarp();
  }

  // ---- share_split of ml (16 bit rows per component) -----------------------
  uint32_t R[3][16];
#pragma unroll
  for (int p = 0; p < 3; ++p) {
    uint32_t a[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const uint32_t v = sm.w32[p][lane * 32 + i] & 0xFFFFu;
      a[i] = v;
    }
    transpose32(a);
#pragma unroll
    for (int j = 0; j < 16; ++j) R[p][j] = a[j];
  }

  // taps (tests only) + start of diff: w32 <- a*ml - b*hd (mod 2^32)
#pragma unroll 4
  for (int i = 0; i < 32; ++i) {
    const int e = lane * 32 + i;
    const uint64_t ln = L0 + e;
    const bool ok = ln >= vb && ln < ve;
#pragma unroll
    for (int p = 0; p < 3; ++p) {
      const uint32_t ml = sm.w32[p][e] & 0xFFFFu;
      const uint32_t hd = sm.s16[p][e];
      if (ok && A.tap_rs_ml) A.tap_rs_ml[p * n + ln] = (uint16_t)ml;
      if (ok && A.tap_rs_hd) A.tap_rs_hd[p * n + ln] = (uint16_t)hd;
      if (ok && A.tap_ml32) A.tap_ml32[p * n + ln] = ml;
      sm.w32[p][e] = A.a * ml - A.b * hd;
    }
  }
  __syncwarp();

  // ---- lift: bits 16 and 17 of x1 + x2 + x3 ---------------------------------
  uint32_t b16[3], b17[3];
  {
    uint64_t base[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) base[k] = A.pos[k] + 2 * n;
    extract_bit<16, 16>(sm, A, base, w0, lane, R, 0, 33, 2, 63, b16);
    extract_bit<17, 16>(sm, A, base, w0, lane, R, 16, 34, 2, 63, b17);
  }

  // ---- bit_inject<15>(bit17), bit_inject<16>(bit16), const-lifted into diff --
#pragma unroll 1
  for (int which = 0; which < 2; ++which) {
    const uint32_t* bits = which == 0 ? b17 : b16;
    const uint32_t mask = which == 0 ? 0x7FFFu : 0xFFFFu;
    const int shift = which == 0 ? 17 : 16;
    const uint64_t o1 = A.pos[0] + 2 * n + 64 * W + (which == 0 ? 0 : n);
    const uint64_t o3 = A.pos[2] + 2 * n + 64 * W + (which == 0 ? 0 : 3 * n);
    warp_fill16(A.key[0], o1 + L0, 1024, 1, sm.s16[0], lane);
    warp_fill16(A.key[2], o3 + 3 * L0, 1024, 3, sm.s16[1], lane);
#pragma unroll 4
    for (int i = 0; i < 32; ++i) {
      const int e = lane * 32 + i;
      const uint32_t x = ((bits[0] ^ bits[1] ^ bits[2]) >> i) & 1u;
      const uint32_t c1 = sm.s16[0][e] & mask;
      const uint32_t c3 = sm.s16[1][e] & mask;
      const uint32_t c2 = (x - c1 - c3) & mask;
      sm.w32[0][e] -= A.a * (c1 << shift);
      sm.w32[1][e] -= A.a * (c2 << shift);
      sm.w32[2][e] -= A.a * (c3 << shift);
      if (A.tap_ml32) {
        const uint64_t ln = L0 + e;
        if (ln >= vb && ln < ve) {
          A.tap_ml32[0 * n + ln] -= c1 << shift;
          A.tap_ml32[1 * n + ln] -= c2 << shift;
          A.tap_ml32[2 * n + ln] -= c3 << shift;
        }
      }
    }
    __syncwarp();
  }

  // ---- msb<32> of diff --------------------------------------------------------
  uint32_t D[3][32];
#pragma unroll
  for (int p = 0; p < 3; ++p) {
#pragma unroll
    for (int i = 0; i < 32; ++i) D[p][i] = sm.w32[p][lane * 32 + i];
    if (A.tap_diff) {
      for (int i = 0; i < 32; ++i) {
        const uint64_t ln = L0 + lane * 32 + i;
        if (ln >= vb && ln < ve) A.tap_diff[p * n + ln] = D[p][i];
      }
    }
    transpose32(D[p]);
  }
  uint32_t bit[3];
  {
    uint64_t base[3];
    base[0] = A.pos[0] + 4 * n + 64 * W;
    base[1] = A.pos[1] + 2 * n + 64 * W;
    base[2] = A.pos[2] + 8 * n + 64 * W;
    extract_bit<31, 32>(sm, A, base, w0, lane, D, 0, 31, 1, 60, bit);
  }

  // ---- outputs ------------------------------------------------------------------
  const uint64_t Lt = L0 + 32ull * lane;
  uint32_t vm = 0;
  if (ve > Lt && vb < Lt + 32) {
    const uint32_t from = vb > Lt ? (uint32_t)(vb - Lt) : 0u;
    const uint32_t to = ve < Lt + 32 ? (uint32_t)(ve - Lt) : 32u;
    vm = (to >= 32 ? 0xFFFFFFFFu : ((1u << to) - 1)) & ~((1u << from) - 1);
  }
#pragma unroll
  for (int c = 0; c < 3; ++c) bit[c] &= vm;
  if (A.tap_msb) {
    for (int i = 0; i < 32; ++i)
      if ((vm >> i) & 1)
        for (int c = 0; c < 3; ++c) A.tap_msb[c * n + Lt + i] = (bit[c] >> i) & 1;
  }
  if (A.match[0]) {
    const uint64_t wi = Lt / 32 - A.match_w0;
    if (vm) {
#pragma unroll
      for (int c = 0; c < 3; ++c) atomicOr(&A.match[c][wi], bit[c]);
    }
  }

  if (sg.slot >= 0) {
    // fused first OR level: 36 AND gates per warp, stream id 1
    uint64_t* orr = &sm.gr[0][0][0];  // [3][40]
    const uint64_t E0 = A.or_elem_base + task * 64;
    __syncwarp();
    for (int s = lane; s < 18; s += 32) {
      const int k = s / 6, bo = s % 6;
      const uint64_t b = E0 / 8 + bo;
      if (b > (E0 + 35) / 8) continue;
      uint32_t blk[16];
      chacha12_block(A.key[k], b, 1, blk);
      for (int w = 0; w < 8; ++w) {
        const uint64_t e = b * 8 + w;
        if (e >= E0 && e < E0 + 36) orr[k * 40 + (e - E0)] = chacha_word(blk, w);
      }
    }
    __syncwarp();
    uint32_t x[3] = {bit[0], bit[1], bit[2]};
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      uint32_t y[3], f[3], z[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) y[c] = __shfl_down_sync(0xffffffffu, x[c], o);
      const int gid = min(32 - 2 * o + lane, 30);
#pragma unroll
      for (int k = 0; k < 3; ++k) f[k] = (uint32_t)orr[k * 40 + gid];
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
        for (int k = 0; k < 3; ++k) f[k] = (uint32_t)orr[k * 40 + 31 + lvl] & m;
        and3(lo_, hi_, f, z);
#pragma unroll
        for (int c = 0; c < 3; ++c) x[c] = lo_[c] ^ hi_[c] ^ (z[c] & m);
      }
      const uint64_t slot = (uint64_t)sg.slot + (task - sg.task_begin);
#pragma unroll
      for (int c = 0; c < 3; ++c) A.partial[c * A.nslots + slot] = (uint8_t)(x[c] & 1u);
    }
  }
}

void launch_threshold(const ThrArgs& a, cudaStream_t st) {
  if (!a.ntasks) return;
  static bool attr = false;
  const int smem = kWarps * (int)sizeof(WarpSmem);
  if (!attr) {
    cudaFuncSetAttribute(k_threshold, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  const unsigned blocks = (unsigned)((a.ntasks + kWarps - 1) / kWarps);
  k_threshold<<<blocks, kWarps * 32, smem, st>>>(a);
}

}  // namespace irisgpu
