// ChaCha12 roofline probe for the threshold phase: the device's pure
// keystream rate with the repo's own chacha12_block (csrc/common.cuh) and the
// k_gate_keystream store pattern (four 16-byte stores per block), plus a
// no-store variant.  ChaCha12 is 48 quarter rounds of 4 add / 4 xor / 4 rotate;
// the xor and rotate (LOP3, SHF) issue on the ALU pipe, so this rate is the
// ALU-pipe ceiling every PRF-consuming threshold kernel is measured against.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -I paper_2405_04463_b200/csrc \
//        tools/chacha_peak.cu -o tools/chacha_peak && tools/chacha_peak
#include <cstdio>
#include <cstdint>

#include "common.cuh"

using namespace irisgpu;

template <bool STORE>
__global__ void __launch_bounds__(256) k_probe(SeedKey key, uint64_t nblk, uint4* out, uint32_t* sink) {
  const uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (b >= nblk) return;
  uint32_t blk[16];
  chacha12_block(key, b, 0, blk);
  if (STORE) {
#pragma unroll
    for (int q = 0; q < 4; ++q) out[4 * b + q] = make_uint4(blk[4 * q], blk[4 * q + 1], blk[4 * q + 2], blk[4 * q + 3]);
  } else {
    uint32_t x = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) x ^= blk[i];
    if (x == 0x9e3779b9u) sink[0] = x;  // keeps the block live
  }
}

template <bool STORE>
static double rate(SeedKey key, uint64_t nblk, uint4* out, uint32_t* sink) {
  const unsigned grid = (unsigned)((nblk + 255) / 256);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  double best = 1e30;
  for (int r = 0; r < 8; ++r) {
    cudaEventRecord(e0);
    k_probe<STORE><<<grid, 256>>>(key, nblk, out, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (r > 1 && ms < best) best = ms;  // two warm-up launches
  }
  return nblk / (best / 1e3);
}

int main() {
  const uint64_t nblk = 1ull << 26;  // 4 GiB of keystream: larger than L2
  uint4* out = nullptr;
  uint32_t* sink = nullptr;
  if (cudaMalloc(&out, nblk * 64) != cudaSuccess || cudaMalloc(&sink, 4) != cudaSuccess) return 1;
  const SeedKey key{{0x0dc1b79bu, 0xfd711811u, 0xbff2b5d4u, 0x8d0deeb1u}};
  const double s = rate<true>(key, nblk, out, sink);
  const double n = rate<false>(key, nblk, out, sink);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  std::printf("{\"chacha12_blocks_per_s_store\": %.4g, \"chacha12_blocks_per_s_nostore\": %.4g, "
              "\"store_GBps\": %.1f, \"blocks\": %llu, \"sm_clock_attr_mhz\": %d, \"error\": \"%s\"}\n",
              s, n, s * 64 / 1e9, (unsigned long long)nblk, clk / 1000, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
