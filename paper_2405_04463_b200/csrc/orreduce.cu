// K5 for DB-sharded queries: bucketed MPC OR-reduction to one shared bit per
// person per shard, the cross-shard OR, and the open at P1 (open_bits_to,
// circuits.hpp:449-486; k_or_open also opens the share-exact tree of
// ortree.cu, which every unsharded query uses).  x OR y = x ^ y ^ (x AND y),
// every AND a 3-party gate with fresh zero-shared randomness from its own
// ChaCha stream ids (or_stream_id).  The reference has no sharded query, so
// this tree shape (buckets per warp task, per person, per shard) has no
// reference shares to match; the opened bit is the same OR.  Partial
// aggregates are never opened (OpenAudit semantics, rep3.hpp:131-134).
#include "common.cuh"
#include "kernels.h"

namespace irisgpu {

namespace {

__device__ __forceinline__ void or_bit(uint32_t acc[3], const uint32_t x[3], const uint32_t f[3]) {
  uint32_t z[3];
#pragma unroll
  for (int p = 0; p < 3; ++p) {
    const int q = (p + 2) % 3;
    z[p] = (acc[p] & x[p]) ^ (acc[q] & x[p]) ^ (acc[p] & x[q]) ^ f[p] ^ f[q];
  }
#pragma unroll
  for (int p = 0; p < 3; ++p) acc[p] = (acc[p] ^ x[p] ^ z[p]) & 1u;
}

__device__ __forceinline__ void rand_elem(const SeedKey* key, uint64_t stream, uint64_t e, uint32_t f[3]) {
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    uint32_t blk[16];
    chacha12_block(key[k], e / 8, stream, blk);
    f[k] = blk[2 * (e % 8)];
  }
}

__device__ __forceinline__ uint64_t pair_index(uint32_t i, uint32_t j, uint32_t persons) {
  return (uint64_t)i * persons - (uint64_t)i * (i + 1) / 2 + (j - i - 1);
}

}  // namespace

__global__ void __launch_bounds__(256) k_or_persons(const OrArgs A) {
  const uint32_t P = blockIdx.x;
  const uint64_t sb = A.slot_begin[P], se = A.slot_begin[P + 1];
  const uint64_t nslot = se - sb;
  const uint64_t npair = A.pair_match[0] ? (uint64_t)(A.persons - 1) * 4 * A.rot : 0;
  const uint64_t nitems = nslot + npair;
  const uint64_t ebase = (uint64_t)P << kOrPersonShift;
  uint32_t acc[3] = {0, 0, 0};
  for (uint64_t c = threadIdx.x; c * 8 < nitems; c += blockDim.x) {
    uint32_t blk[3][16];
#pragma unroll
    for (int k = 0; k < 3; ++k) chacha12_block(A.key[k], ebase / 8 + c, A.stream, blk[k]);
    for (int w = 0; w < 8; ++w) {
      const uint64_t u = c * 8 + w;
      if (u >= nitems) break;
      uint32_t x[3];
      if (u < nslot) {
#pragma unroll
        for (int k = 0; k < 3; ++k) x[k] = A.partial[k * A.nslots + sb + u] & 1u;
      } else {
        const uint64_t up = u - nslot;
        const uint32_t qi = (uint32_t)(up / (4ull * A.rot));
        const uint32_t Q = qi < P ? qi : qi + 1;
        const uint32_t i = P < Q ? P : Q, j = P < Q ? Q : P;
        const uint64_t pl = pair_index(i, j, A.persons) * 4ull * A.rot + up % (4ull * A.rot);
        const uint64_t gl = A.pair_lane0 + pl;
        const uint64_t wi = gl / 32 - A.pair_w0;
#pragma unroll
        for (int k = 0; k < 3; ++k) x[k] = (A.pair_match[k][wi] >> (gl % 32)) & 1u;
      }
      uint32_t f[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) f[k] = blk[k][2 * w];
      or_bit(acc, x, f);
    }
  }
  // block tree: warp shuffles, then across the 8 warps
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t tb = ebase + kOrTreeOffset;
  for (int o = 16; o >= 1; o >>= 1) {
    uint32_t y[3], f[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) y[k] = __shfl_down_sync(0xffffffffu, acc[k], o);
    rand_elem(A.key, A.stream, tb + (uint64_t)(5 - __ffs(o)) * 256 + threadIdx.x, f);
    if (lane < o) or_bit(acc, y, f);
  }
  __shared__ uint32_t wsum[8][3];
  if (lane == 0)
    for (int k = 0; k < 3; ++k) wsum[warp][k] = acc[k];
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t r[3] = {wsum[0][0], wsum[0][1], wsum[0][2]};
    for (int w = 1; w < (int)(blockDim.x / 32); ++w) {
      uint32_t f[3];
      rand_elem(A.key, A.stream, tb + 5 * 256 + w, f);
      or_bit(r, wsum[w], f);
    }
    for (int k = 0; k < 3; ++k) A.out[k * A.persons + P] = (uint8_t)r[k];
  }
}

// Final OR over G shard partials [G][3][persons] and the open at P1
// (open_bits_to, circuits.hpp:449-486).  In this co-resident component form each
// XOR component exists once, so P1's cross-check of the two copies of component
// 2 (circuits.hpp:470-472) has nothing to compare; party mode (party.cu), where
// P2 and P3 really send their copies, performs it.
__global__ void k_or_open(const uint8_t* __restrict__ partials, uint32_t G, uint32_t persons,
                          SeedKey k1, SeedKey k2, SeedKey k3, uint64_t stream, uint8_t* match) {
  const uint32_t P = blockIdx.x * blockDim.x + threadIdx.x;
  if (P >= persons) return;
  const SeedKey key[3] = {k1, k2, k3};
  uint32_t acc[3];
  for (int k = 0; k < 3; ++k) acc[k] = partials[k * persons + P] & 1u;
  for (uint32_t g = 1; g < G; ++g) {
    uint32_t x[3], f[3];
    for (int k = 0; k < 3; ++k) x[k] = partials[((uint64_t)g * 3 + k) * persons + P] & 1u;
    rand_elem(key, stream, ((uint64_t)P << 32) + g, f);
    or_bit(acc, x, f);
  }
  match[P] = (uint8_t)((acc[0] ^ acc[1] ^ acc[2]) & 1u);
}

void launch_or_persons(const OrArgs& a, cudaStream_t st) {
  if (!a.persons) return;
  k_or_persons<<<a.persons, 256, 0, st>>>(a);
}

void launch_or_open(const uint8_t* partials, uint32_t G, uint32_t persons, const SeedKey key[3],
                    uint64_t stream, uint8_t* match_out, cudaStream_t st) {
  if (!persons) return;
  k_or_open<<<(persons + 127) / 128, 128, 0, st>>>(partials, G, persons, key[0], key[1], key[2],
                                                     stream, match_out);
}

}  // namespace irisgpu
