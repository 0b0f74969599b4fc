// ChaCha12 load generator for tools/energy_query.py --corun: the repo's
// chacha12_block (csrc/common.cuh) as a grid-stride kernel behind a C entry
// point, so a pure-ALU keystream of a given size and footprint can run on a
// second stream next to a query.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -shared \
//        -I paper_2405_04463_b200/csrc tools/chacha_launch.cu -o tools/_build/libchacha_launch.so
#include <cstdint>
#include <cuda_runtime.h>

#include "common.cuh"

using namespace irisgpu;

__global__ void __launch_bounds__(256) k_chacha_load(SeedKey key, uint64_t b0, uint64_t nblk, uint32_t* sink) {
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < nblk; t += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t blk[16];
    chacha12_block(key, b0 + t, 0, blk);
    uint32_t x = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) x ^= blk[i];
    if (x == 0x9e3779b9u) sink[0] = x;  // keeps the block live, no memory traffic
  }
}

// grid = 0: one thread per block; threads = 0: 256
extern "C" int chacha_load(void* stream, uint64_t nblk, uint64_t b0, unsigned grid, unsigned threads, void* sink) {
  const SeedKey key{{1, 2, 3, 4}};
  if (!threads) threads = 256;
  if (!grid) grid = (unsigned)((nblk + threads - 1) / threads);
  k_chacha_load<<<grid, threads, 0, (cudaStream_t)stream>>>(key, b0, nblk, (uint32_t*)sink);
  return (int)cudaGetLastError();
}
