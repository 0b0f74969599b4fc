// Inner-batch pair lanes: the rotated eye of person i against the centre eye
// of every later person j (engine.cpp:275-293, detail::rep_pair_dot /
// gr_pair_dot engine.hpp:208-219).  These are 0.003% of the lanes at the
// headline configs, so they run as a plain warp-per-dot kernel; the DB lanes
// go through the tcgen05 GEMM.
#include "common.cuh"
#include "kernels.h"

namespace irisgpu {

__global__ void k_pairs(const uint16_t* __restrict__ pa, const uint16_t* __restrict__ pb,
                        uint32_t ncodes, uint32_t persons, uint32_t l, uint32_t rot, int shamir,
                        uint64_t npairs, uint16_t* __restrict__ out_hd, uint16_t* __restrict__ out_ml,
                        uint64_t out_pstride) {
  const uint64_t wid = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (wid >= npairs * 6) return;
  const uint64_t k = wid / 6;
  const int prob = (int)(wid % 6);  // p * 2 + d
  // decode k = pair_index(i, j) * 4r + ea * 2r + eb * r + rot_j
  const uint32_t rr = (uint32_t)(k % rot);
  uint64_t t = k / rot;
  const uint32_t eb = (uint32_t)(t % 2);
  t /= 2;
  const uint32_t ea = (uint32_t)(t % 2);
  uint64_t pidx = t / 2;
  uint32_t i = 0;
  while (pidx >= persons - 1 - i) {
    pidx -= persons - 1 - i;
    ++i;
  }
  const uint32_t j = i + 1 + (uint32_t)pidx;
  const uint32_t half = (rot - 1) / 2;
  const int64_t by = ((int64_t)rr - (int64_t)half) * (int64_t)(l / 64);
  const uint64_t xbase = ((uint64_t)prob * ncodes + 2 * i + ea) * l;
  const uint64_t ybase = ((uint64_t)prob * ncodes + 2 * j + eb) * l;
  uint32_t acc = 0;
  // rotated index src = (kk - by) mod len, advanced by 32 with a conditional wrap
  if (shamir) {
    const uint32_t h = l / 2;
    int64_t bp = (by / 2) % (int64_t)h;
    if (bp < 0) bp += h;
    for (uint32_t seg = 0; seg < l; seg += h) {
      uint32_t src = (uint32_t)((lane + h - (uint32_t)bp) % h);
      for (uint32_t kk = lane; kk < h; kk += 32) {
        acc += (uint32_t)pa[xbase + seg + src] * (uint32_t)pb[ybase + seg + kk];
        src += 32;
        while (src >= h) src -= h;
      }
    }
  } else {
    int64_t b0 = by % (int64_t)l;
    if (b0 < 0) b0 += l;
    uint32_t src = (uint32_t)((lane + l - (uint32_t)b0) % l);
    for (uint32_t kk = lane; kk < l; kk += 32) {
      acc += (uint32_t)pa[xbase + src] * (uint32_t)pa[ybase + kk];
      acc -= (uint32_t)pb[xbase + src] * (uint32_t)pb[ybase + kk];
      src += 32;
      while (src >= l) src -= l;
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) {
    uint16_t* out = (prob & 1) ? out_ml : out_hd;
    out[(uint64_t)(prob >> 1) * out_pstride + k] = (uint16_t)acc;
  }
}

void launch_pairs(const uint16_t* pa, const uint16_t* pb, uint32_t ncodes, uint32_t persons,
                  uint32_t l, uint32_t rot, int shamir, uint16_t* out_hd, uint16_t* out_ml,
                  uint64_t out_pstride, cudaStream_t st) {
  if (persons < 2) return;
  const uint64_t npairs = (uint64_t)persons * (persons - 1) / 2 * 4 * rot;
  const uint64_t threads = npairs * 6 * 32;
  const unsigned blocks = (unsigned)((threads + 255) / 256);
  k_pairs<<<blocks, 256, 0, st>>>(pa, pb, ncodes, persons, l, rot, shamir, npairs, out_hd, out_ml,
                                  out_pstride);
}

}  // namespace irisgpu
