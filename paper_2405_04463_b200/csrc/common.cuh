// Shared device helpers for the B200 irismpc hot path (sm_100a only).
//
//  * ChaCha12 counter PRF, bit-compatible with the reference CtrPrf
//    (/root/reference/proj/include/irismpc/prf.hpp:46-135): stream element
//    idx is u64 word idx%8 of block idx/8.
//  * Thin inline-PTX wrappers for mbarrier / TMA / tcgen05.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "irismpc_b200 targets sm_100a only"
#endif

namespace irisgpu {

// ---------------------------------------------------------------- ChaCha12

struct SeedKey {
  uint32_t k[4];
};

__host__ __device__ __forceinline__ uint32_t rotl(uint32_t x, int n) {
#ifdef __CUDA_ARCH__
  return __funnelshift_l(x, x, n);
#else
  return (x << n) | (x >> (32 - n));
#endif
}

#define IRIS_QR(a, b, c, d)          \
  a += b; d ^= a; d = rotl(d, 16);   \
  c += d; b ^= c; b = rotl(b, 12);   \
  a += b; d ^= a; d = rotl(d, 8);    \
  c += d; b ^= c; b = rotl(b, 7);

// detail::chacha_block (prf.hpp:46-69): key duplicated into words 4..11,
// 64-bit block counter in 12..13, 64-bit stream id in 14..15, 12 rounds.
__host__ __device__ __forceinline__ void chacha12_block(const SeedKey& key, uint64_t block,
                                                        uint64_t stream, uint32_t out[16]) {
  const uint32_t c0 = 0x61707865u, c1 = 0x3320646eu, c2 = 0x79622d32u, c3 = 0x6b206574u;
  uint32_t x0 = c0, x1 = c1, x2 = c2, x3 = c3;
  uint32_t x4 = key.k[0], x5 = key.k[1], x6 = key.k[2], x7 = key.k[3];
  uint32_t x8 = key.k[0], x9 = key.k[1], x10 = key.k[2], x11 = key.k[3];
  uint32_t x12 = (uint32_t)block, x13 = (uint32_t)(block >> 32);
  uint32_t x14 = (uint32_t)stream, x15 = (uint32_t)(stream >> 32);
#pragma unroll
  for (int r = 0; r < 6; ++r) {
    IRIS_QR(x0, x4, x8, x12);
    IRIS_QR(x1, x5, x9, x13);
    IRIS_QR(x2, x6, x10, x14);
    IRIS_QR(x3, x7, x11, x15);
    IRIS_QR(x0, x5, x10, x15);
    IRIS_QR(x1, x6, x11, x12);
    IRIS_QR(x2, x7, x8, x13);
    IRIS_QR(x3, x4, x9, x14);
  }
  out[0] = x0 + c0; out[1] = x1 + c1; out[2] = x2 + c2; out[3] = x3 + c3;
  out[4] = x4 + key.k[0]; out[5] = x5 + key.k[1]; out[6] = x6 + key.k[2]; out[7] = x7 + key.k[3];
  out[8] = x8 + key.k[0]; out[9] = x9 + key.k[1]; out[10] = x10 + key.k[2]; out[11] = x11 + key.k[3];
  out[12] = x12 + (uint32_t)block; out[13] = x13 + (uint32_t)(block >> 32);
  out[14] = x14 + (uint32_t)stream; out[15] = x15 + (uint32_t)(stream >> 32);
}

__host__ __device__ __forceinline__ uint64_t chacha_word(const uint32_t blk[16], int w) {
  return (uint64_t)blk[2 * w] | ((uint64_t)blk[2 * w + 1] << 32);
}

// ---------------------------------------------------------------- PTX

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t"
      ".reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@P1 bra DONE_%=;\n\t"
      "bra WAIT_%=;\n\t"
      "DONE_%=:\n\t"
      "}" ::"r"(smem_u32(bar)),
      "r"(phase), "r"(0x989680)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const void* tmap, uint64_t* bar, int32_t c0,
                                            int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

__device__ __forceinline__ void tma_prefetch_desc(const void* tmap) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(tmap) : "memory");
}

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// tcgen05.commit: arrive on an mbarrier once all prior MMAs of this thread finish.
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

// D[tmem] (+)= A[smem] * B[smem]^T, u8 x u8 -> s32, cta_group::1.
__device__ __forceinline__ void umma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                        uint32_t idesc, uint32_t accumulate) {
  const uint32_t m0 = 0, m1 = 0, m2 = 0, m3 = 0;
  asm volatile(
      "{\n\t"
      ".reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, {%5, %6, %7, %8}, p;\n\t"
      "}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(m0), "r"(m1), "r"(m2), "r"(m3));
}

// ---- CTA-pair (cta_group::2) variants -------------------------------------
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// one lane of a converged warp (the issue lane of TMA / tcgen05.mma): keeping the
// producer and MMA loops warp-uniform lets their descriptor and coordinate math
// live in uniform registers (uniform datapath) instead of the vector ALU pipe,
// which the co-resident ChaCha kernels saturate
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of `p` in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa_shared(const void* p, uint32_t rank) {
  uint32_t out;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(out) : "r"(smem_u32(p)), "r"(rank));
  return out;
}
// arrive (release, cluster scope) on an mbarrier given by its cluster address
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t bar_cluster) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster) : "memory");
}
// TMA load into this CTA's smem, completion bytes counted on the barrier at
// cluster address bar_cluster (the leader CTA's full barrier).
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const void* tmap, uint32_t bar_cluster, int32_t c0,
                                                 int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(bar_cluster), "r"(c0), "r"(c1)
      : "memory");
}
// commit prior cta_group::2 MMAs to the same-offset barrier in every CTA of mask
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}
__device__ __forceinline__ void umma_i8_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                             uint32_t accumulate) {
  const uint32_t z = 0;
  asm volatile(
      "{\n\t"
      ".reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, {%5, %5, %5, %5, %5, %5, %5, %5}, p;\n\t"
      "}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(z));
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
      "%12, %13, %14, %15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}

__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// ------------------------------------------------------ bit-slice helpers

// In-place 32x32 bit-matrix transpose: on return bit i of a[j] equals bit j
// of the input a[i] (rows = lanes in, rows = bit planes out).
__host__ __device__ __forceinline__ void transpose32(uint32_t (&a)[32]) {
  uint32_t m = 0x0000FFFFu;
#pragma unroll
  for (int j = 16; j != 0; j >>= 1, m ^= (m << j)) {
#pragma unroll
    for (int k = 0; k < 32; k = ((k | j) + 1) & ~j) {
      const uint32_t t = ((a[k] >> j) ^ a[k | j]) & m;
      a[k] ^= t << j;
      a[k | j] ^= t;
    }
  }
}

// ---- warp-cooperative stream windows.  The lane-major kernels map 31
// consecutive 8-lane groups to a warp (lane 31 only helps).  A lane's window
// of 8 * NB elements starting at e spans NB blocks + 1 when e % 8 != 0
// (warp-uniform: e = stream offset + 8 * group); the extra block is the next
// lane's first block and arrives by shuffle, so every ChaCha block is
// computed once instead of up to twice.  Only the low 32 bits of each u64
// element are consumed (Ring<K <= 32> draws).
template <int NB, int R>
__device__ __forceinline__ void take_window(const uint32_t (&w)[8 * (NB + 1)], uint32_t (&out)[8 * NB]) {
#pragma unroll
  for (int i = 0; i < 8 * NB; ++i) out[i] = w[R + i];
}

// next_contig: lane + 1 owns the window starting at e + 8 * NB (else this lane
// computes the extra block itself -- segment boundaries, the last group).
// Must be called by all 32 lanes in convergent code.
template <int NB>
__device__ __forceinline__ void prf_window(const SeedKey& key, uint64_t e, bool next_contig,
                                           uint32_t (&out)[8 * NB]) {
  uint32_t w[8 * (NB + 1)];
  const uint64_t b = e / 8;
#pragma unroll
  for (int q = 0; q < NB; ++q) {
    uint32_t blk[16];
    chacha12_block(key, b + q, 0, blk);
#pragma unroll
    for (int i = 0; i < 8; ++i) w[8 * q + i] = blk[2 * i];
  }
  const int r = (int)(e % 8);
  if (r == 0) {
#pragma unroll
    for (int i = 0; i < 8 * NB; ++i) out[i] = w[i];
    return;
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) w[8 * NB + i] = __shfl_down_sync(0xFFFFFFFFu, w[i], 1);
  if (!next_contig) {
    uint32_t blk[16];
    chacha12_block(key, b + NB, 0, blk);
#pragma unroll
    for (int i = 0; i < 8; ++i) w[8 * NB + i] = blk[2 * i];
  }
  switch (r) {
    case 1: take_window<NB, 1>(w, out); break;
    case 2: take_window<NB, 2>(w, out); break;
    case 3: take_window<NB, 3>(w, out); break;
    case 4: take_window<NB, 4>(w, out); break;
    case 5: take_window<NB, 5>(w, out); break;
    case 6: take_window<NB, 6>(w, out); break;
    default: take_window<NB, 7>(w, out); break;
  }
}

}  // namespace irisgpu
