// Lane-major reshare / bit-inject (the round-1 kernels: thread = 8 lanes,
// warp-cooperative ChaCha windows), kept as an A/B alternative to the
// 512-lane tile kernels of threshold.cu (IRISMPC_THR_KERNELS=tile|lm).  Same semantics
// (reshare_pair, engine.cpp:80-106; bit_inject, convert.hpp:84-155).
#include <type_traits>

#include "common.cuh"
#include "kernels.h"

namespace irisgpu {

namespace {

// lane -> 8-lane group of a lane-major kernel (31 groups per warp)
struct GroupCtx {
  uint64_t L8;       // first global lane of the group
  bool mine;         // this lane owns a real group (lane < 31, group < ngrp)
  bool next_contig;  // lane + 1 owns the group at L8 + 8
  const Seg* sg;
};

// 3-D grids: blockIdx.z = segment, so no search; warp w of block x owns the
// segment's 8-lane groups [(x * warps + w) * 31, + 31).  Returns false when the
// whole warp lies past the segment (warp-uniform).
__device__ __forceinline__ bool group_ctx(const ThrArgs& A, GroupCtx& c) {
  const int lane = threadIdx.x & 31;
  c.sg = &A.segs[blockIdx.z];
  const uint64_t g0 = c.sg->lane_begin / 8;
  const uint64_t ng = (c.sg->lane_end - 1) / 8 - g0 + 1;
  const uint64_t w0 = ((uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 31;
  if (w0 >= ng) return false;
  const uint64_t gi = w0 + lane;
  c.mine = lane < 31 && gi < ng;
  c.L8 = (g0 + (gi < ng ? gi : ng - 1)) * 8;
  c.next_contig = lane == 31 || gi + 1 < ng;
  return true;
}



// 8 lanes [L8, L8+8) of a dot array (u16 or u32) -> v[0..7]; `full`: one aligned vector access
template <typename T>
__device__ __forceinline__ void load8_at(const T* src, uint64_t src0, const Seg& sg, uint64_t L8, bool full,
                                         bool mine, uint32_t v[8]) {
  if (full) {
    if (sizeof(T) == 2) {
      const uint4 x = *reinterpret_cast<const uint4*>(src + src0);
      const uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        v[2 * i] = w[i] & 0xFFFFu;
        v[2 * i + 1] = w[i] >> 16;
      }
    } else {
      const uint4 x = reinterpret_cast<const uint4*>(src + src0)[0];
      const uint4 y = reinterpret_cast<const uint4*>(src + src0)[1];
      v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
      v[4] = y.x; v[5] = y.y; v[6] = y.z; v[7] = y.w;
    }
    return;
  }
  const uint64_t base = src0 - (L8 - sg.lane_begin);  // index of lane_begin
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint64_t ln = L8 + i;
    const bool ok = mine && ln >= sg.lane_begin && ln < sg.lane_end;
    v[i] = ok ? (uint32_t)src[base + (ln - sg.lane_begin)] : 0u;
  }
}

// A field's dots of lanes [L8, L8+8): plain [col][row] planes, or (RP) the sum
// of the rotation pair's shared product P2 and its own P1 / P3 (prep.cu)
template <typename T>
__device__ __forceinline__ void load8(const T* src, uint64_t kstride, const Seg& sg, uint64_t L8, bool full,
                                      bool mine, uint32_t v[8]) {
  if (!kstride) {
    load8_at<T>(src, sg.src + (L8 - sg.lane_begin), sg, L8, full, mine, v);
    return;
  }
  const uint64_t i0 = sg.src_rp + (L8 - sg.lane_begin);
  uint32_t a[8];
  load8_at<T>(src, i0 + kstride, sg, L8, full, mine, v);
  load8_at<T>(src, i0 + (sg.rp_sel == 1 ? 0 : 2 * kstride), sg, L8, full, mine, a);
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] += a[i];
}

// reshare one dot (zero_ring<K>, rep3.hpp:110-112): component k gains F_k and
// component k+1 loses it -- own_p = z_p + F(seed_p) - F(seed_{p-1})
__device__ __forceinline__ void reshare8(const ThrArgs& A, uint64_t e_off, bool next_contig, uint32_t v[3][8],
                                         uint32_t kmask) {
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    uint32_t f[8];
    prf_window<1>(A.key[k], A.pos[k] + e_off, next_contig, f);
    const int kn = (k + 1) % 3;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      v[k][i] += f[i];
      v[kn][i] -= f[i];
    }
  }
#pragma unroll
  for (int p = 0; p < 3; ++p)
#pragma unroll
    for (int i = 0; i < 8; ++i) v[p][i] &= kmask;
}


}  // namespace


// thread -> 8-lane group (global lane multiple of 8) of one segment.
// reshare_pair<KH, KM> (engine.cpp:80-106: hd lanes at stream offset 0, ml at
// n) followed by the comparison input:
//   mpc-lift   : ml_rs = ml (u16, lifted later), diff = a ml - b hd (partial)
//   const-lift : diff = a ml32 - const_lift(hd, b)      (engine.hpp:94-120)
//   no-lift    : diff = a ml32 - b hd32
//   plain-mask : diff = public_minus(ceil((1-2r) ml), hd) (engine.hpp:77-90)
template <int V>
#ifndef RESHARE_LM_MINB
#define RESHARE_LM_MINB 2  // min CTAs per SM (register cap), A/B: -DRESHARE_LM_MINB=n
#endif
#ifndef INJECT_LM_MINB
#define INJECT_LM_MINB 1
#endif
__global__ void __launch_bounds__(256, RESHARE_LM_MINB) k_reshare_lm(const __grid_constant__ ThrArgs A) {
  using HT = typename std::conditional<V == kNoLift, uint32_t, uint16_t>::type;
  using MT = typename std::conditional<V == kConstLift || V == kNoLift, uint32_t, uint16_t>::type;
  constexpr uint32_t HM = V == kNoLift ? 0xFFFFFFFFu : 0xFFFFu;
  constexpr uint32_t MM = (V == kConstLift || V == kNoLift) ? 0xFFFFFFFFu : 0xFFFFu;
  GroupCtx gc;
  if (!group_ctx(A, gc)) return;  // whole warp past the segment
  const Seg& sg = *gc.sg;
  const uint64_t L8 = gc.L8;
  const uint64_t src0 = sg.src + (L8 - sg.lane_begin);  // valid only when `full`
  bool full = gc.mine && L8 >= sg.lane_begin && L8 + 8 <= sg.lane_end && !A.tap_rs_hd;
  const HT* hd[3];
  const MT* ml[3];
  const uint64_t rp0 = sg.src_rp + (L8 - sg.lane_begin);
  const uint64_t hs0 = A.rp_kstride_h ? rp0 : src0, ms0 = A.rp_kstride_m ? rp0 : src0;
  const uint64_t hk = A.rp_kstride_h, mk = A.rp_kstride_m;
  full = full && hk % 8 == 0 && mk % 8 == 0;  // P2 / P3 vectors stay 16-byte aligned
#pragma unroll
  for (int p = 0; p < 3; ++p) {
    hd[p] = static_cast<const HT*>(A.hd[p]);
    ml[p] = static_cast<const MT*>(A.ml[p]);
    // 16-byte alignment of every vector access (RP: all three P planes; kstride is a multiple of 8)
    full = full && ((reinterpret_cast<uintptr_t>(hd[p] + hs0) | reinterpret_cast<uintptr_t>(ml[p] + ms0) |
                     reinterpret_cast<uintptr_t>(A.diff + p * A.cstride + src0)) & 15) == 0;
    if (V == kMpcLift) full = full && (reinterpret_cast<uintptr_t>(A.ml_rs + p * A.cstride + src0) & 15) == 0;
  }
  // ml first (stream offset n): d = a * ml, the reshared ml leaves the registers,
  // then hd (offset 0): d -= b * hd -- keeps two 3 x 8 arrays live, not three
  uint32_t d[3][8], m[3][8];
  if (V != kPlainMask) {
#pragma unroll
    for (int p = 0; p < 3; ++p) load8<MT>(ml[p], mk, sg, L8, full, gc.mine, m[p]);
    if (!A.no_reshare) reshare8(A, A.n + L8, gc.next_contig, m, MM);
#pragma unroll
    for (int p = 0; p < 3; ++p)
#pragma unroll
      for (int i = 0; i < 8; ++i) d[p][i] = A.a * m[p][i];
    if (gc.mine && V == kMpcLift) {
#pragma unroll
      for (int p = 0; p < 3; ++p) {
        if (full) {
          uint32_t mw[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) mw[i] = m[p][2 * i] | (m[p][2 * i + 1] << 16);
          *reinterpret_cast<uint4*>(A.ml_rs + p * A.cstride + src0) = make_uint4(mw[0], mw[1], mw[2], mw[3]);
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const uint64_t ln = L8 + i;
            if (ln >= sg.lane_begin && ln < sg.lane_end)
              A.ml_rs[p * A.cstride + sg.src + (ln - sg.lane_begin)] = (uint16_t)m[p][i];
          }
        }
      }
    }
    if (gc.mine && A.tap_rs_ml) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const uint64_t ln = L8 + i;
        if (ln < sg.lane_begin || ln >= sg.lane_end) continue;
#pragma unroll
        for (int p = 0; p < 3; ++p) {
          A.tap_rs_ml[p * A.n + ln] = m[p][i];
          A.tap_ml32[p * A.n + ln] = m[p][i];
        }
      }
    }
  }
  uint32_t (&h)[3][8] = m;  // reuse the registers
#pragma unroll
  for (int p = 0; p < 3; ++p) load8<HT>(hd[p], hk, sg, L8, full, gc.mine, h[p]);
  if (!A.no_reshare) reshare8(A, L8, gc.next_contig, h, HM);
  if (V == kPlainMask) {
    // public popcount; diff = public_minus(t, hd): component 1 absorbs t (rep3.hpp:59-71)
    uint32_t cnt[8];
    load8<MT>(ml[0], mk, sg, L8, full, gc.mine, cnt);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint32_t t = (uint32_t)(int64_t)ceil(__dmul_rn(A.coef, (double)cnt[i]));
      d[0][i] = (t - h[0][i]) & 0xFFFFu;
      d[1][i] = (0u - h[1][i]) & 0xFFFFu;
      d[2][i] = (0u - h[2][i]) & 0xFFFFu;
    }
  } else {
#pragma unroll
    for (int p = 0; p < 3; ++p)
#pragma unroll
      for (int i = 0; i < 8; ++i) d[p][i] -= A.b * h[p][i];
  }
  if (!gc.mine) return;
  if (full) {
#pragma unroll
    for (int p = 0; p < 3; ++p) {
      uint4* dd = reinterpret_cast<uint4*>(A.diff + p * A.cstride + src0);
      dd[0] = make_uint4(d[p][0], d[p][1], d[p][2], d[p][3]);
      dd[1] = make_uint4(d[p][4], d[p][5], d[p][6], d[p][7]);
    }
    return;
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint64_t ln = L8 + i;
    if (ln < sg.lane_begin || ln >= sg.lane_end) continue;
    const uint64_t src = sg.src + (ln - sg.lane_begin);
#pragma unroll
    for (int p = 0; p < 3; ++p) {
      A.diff[p * A.cstride + src] = d[p][i];
      if (A.tap_rs_hd) A.tap_rs_hd[p * A.n + ln] = h[p][i];
    }
  }
}

// thread -> 8-lane group: bit_inject<15>(bit17) then bit_inject<16>(bit16)
__global__ void __launch_bounds__(256, INJECT_LM_MINB) k_inject_lm(const __grid_constant__ ThrArgs A) {
  GroupCtx gc;
  if (!group_ctx(A, gc)) return;  // whole warp past the segment
  const Seg& sg = *gc.sg;
  const uint64_t L8 = gc.L8;
  // injected bits: the k_lift thread that owns these lanes
  const uint64_t task = sg.task_begin + (L8 / 1024 - sg.q_first);
  const uint64_t o = task * 32 + (L8 % 1024) / 32;
  const int sh = (int)(L8 % 32);
  uint32_t x17 = 0, x16 = 0;
  if (gc.mine) {
    x17 = (A.bits[3 * A.nbits + o] ^ A.bits[4 * A.nbits + o] ^ A.bits[5 * A.nbits + o]) >> sh;
    x16 = (A.bits[0 * A.nbits + o] ^ A.bits[1 * A.nbits + o] ^ A.bits[2 * A.nbits + o]) >> sh;
  }
  uint32_t d[3][8];
  const uint64_t n = A.n;
#pragma unroll
  for (int p = 0; p < 3; ++p)
#pragma unroll
    for (int i = 0; i < 8; ++i) d[p][i] = 0u;
#pragma unroll
  for (int which = 0; which < 2; ++which) {
    const uint32_t x = which == 0 ? x17 : x16;
    const uint32_t mask = which == 0 ? 0x7FFFu : 0xFFFFu;
    const int shift = which == 0 ? 17 : 16;
    const uint64_t o1 = A.inj_base[0] + (which == 0 ? 0 : n) + L8;
    const uint64_t o3 = A.inj_base[2] + (which == 0 ? 0 : 3 * n) + 3 * L8;
    uint32_t c1[8], w3[24];
    prf_window<1>(A.key[0], o1, gc.next_contig, c1);
    prf_window<3>(A.key[2], o3, gc.next_contig, w3);  // (c3, w0, w1) per lane; only c3 is used
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint32_t b1 = c1[i] & mask;
      const uint32_t b3 = w3[3 * i] & mask;
      const uint32_t b2 = (((x >> i) & 1u) - b1 - b3) & mask;
      d[0][i] += b1 << shift;
      d[1][i] += b2 << shift;
      d[2][i] += b3 << shift;
    }
  }
  if (!gc.mine) return;
  const uint64_t src0 = sg.src + (L8 - sg.lane_begin);
  bool vec = L8 >= sg.lane_begin && L8 + 8 <= sg.lane_end && !A.tap_ml32;
#pragma unroll
  for (int p = 0; p < 3; ++p) vec = vec && (reinterpret_cast<uintptr_t>(A.diff + p * A.cstride + src0) & 15) == 0;
  if (vec) {
#pragma unroll
    for (int p = 0; p < 3; ++p) {
      uint4* dd = reinterpret_cast<uint4*>(A.diff + p * A.cstride + src0);
      uint4 x = dd[0], y = dd[1];
      x.x -= A.a * d[p][0]; x.y -= A.a * d[p][1]; x.z -= A.a * d[p][2]; x.w -= A.a * d[p][3];
      y.x -= A.a * d[p][4]; y.y -= A.a * d[p][5]; y.z -= A.a * d[p][6]; y.w -= A.a * d[p][7];
      dd[0] = x;
      dd[1] = y;
    }
    return;
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint64_t ln = L8 + i;
    if (ln < sg.lane_begin || ln >= sg.lane_end) continue;
    const uint64_t src = sg.src + (ln - sg.lane_begin);
#pragma unroll
    for (int p = 0; p < 3; ++p) {
      A.diff[p * A.cstride + src] -= A.a * d[p][i];
      if (A.tap_ml32) A.tap_ml32[p * n + ln] -= d[p][i];
    }
  }
}

void launch_reshare_lm(const ThrArgs& a, cudaStream_t st) {
  const dim3 g((a.grp_seg_max + 8 * 31 - 1) / (8 * 31), 1, a.nsegs);
  switch (a.variant) {
    case kPlainMask: k_reshare_lm<kPlainMask><<<g, 256, 0, st>>>(a); break;
    case kMpcLift: k_reshare_lm<kMpcLift><<<g, 256, 0, st>>>(a); break;
    case kConstLift: k_reshare_lm<kConstLift><<<g, 256, 0, st>>>(a); break;
    default: k_reshare_lm<kNoLift><<<g, 256, 0, st>>>(a); break;
  }
}

void launch_inject_lm(const ThrArgs& a, cudaStream_t st) {
  const dim3 g((a.grp_seg_max + 8 * 31 - 1) / (8 * 31), 1, a.nsegs);
  k_inject_lm<<<g, 256, 0, st>>>(a);
}

}  // namespace irisgpu
