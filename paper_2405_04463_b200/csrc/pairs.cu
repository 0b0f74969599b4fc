// Inner-batch pair lanes: the rotated eye of person i against the centre eye
// of every later person j (engine.cpp:275-293, detail::rep_pair_dot /
// gr_pair_dot engine.hpp:208-219).
//
// They run on the tensor cores as one more limb GEMM: rotating x by +r against
// the centre of y equals x against y rotated by -r, i.e. rotation index
// 2*half - r of the already-built rotated query planes (B).  With A = the
// unrotated query codes parsed exactly like DB rows (Shamir: lambda_p-scaled
// [lc0 | lc1]; replicated: [own | prev] via the component planes), the GEMM
// yields every (x code, y code, rotation) dot; replicated needs the identity
//   sum_x' sum_y - prev_x' prev_y = own_x sum_y'' + prev_x own_y''
// (x' = x rotated by +r, y'' = y rotated by -r), which is exactly the DB-side
// A = [x_p | x_{p-1}], B = [y_p + y_{p-1} | y_p] contraction.  This kernel only
// gathers the needed entries into pair-lane order.
#include "common.cuh"
#include "kernels.h"

namespace irisgpu {

// C: [nprob][ncols][ncodes] (GEMM output, col = code*rot + rotation, row = code)
template <typename T>
__global__ void k_pair_gather(const T* __restrict__ C, uint32_t nprob, uint32_t ncodes, uint32_t ncols,
                              uint32_t persons, uint32_t rot, uint64_t npairs, T* __restrict__ out,
                              uint64_t out_pstride) {
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (tid >= npairs * nprob) return;
  const uint32_t prob = (uint32_t)(tid / npairs);
  const uint64_t k = tid % npairs;  // pair lane: ((pidx * 2 + ea) * 2 + eb) * rot + rr
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
  const uint64_t col = (uint64_t)(2 * j + eb) * rot + (rot - 1 - rr);
  const uint64_t row = 2 * i + ea;
  out[(uint64_t)prob * out_pstride + k] = C[(uint64_t)prob * ncols * ncodes + col * ncodes + row];
}

void launch_pair_gather(const void* C, int elem_bytes, uint32_t nprob, uint32_t ncodes, uint32_t ncols,
                        uint32_t persons, uint32_t rot, void* out, uint64_t out_pstride, cudaStream_t st) {
  if (persons < 2) return;
  const uint64_t npairs = (uint64_t)persons * (persons - 1) / 2 * 4 * rot;
  const unsigned blocks = (unsigned)((npairs * nprob + 255) / 256);
  if (elem_bytes == 4)
    k_pair_gather<uint32_t><<<blocks, 256, 0, st>>>(static_cast<const uint32_t*>(C), nprob, ncodes, ncols, persons,
                                                    rot, npairs, static_cast<uint32_t*>(out), out_pstride);
  else
    k_pair_gather<uint16_t><<<blocks, 256, 0, st>>>(static_cast<const uint16_t*>(C), nprob, ncodes, ncols, persons,
                                                    rot, npairs, static_cast<uint16_t*>(out), out_pstride);
}

}  // namespace irisgpu
