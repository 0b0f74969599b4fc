// K2: Z_2^16 share dot products as u8-limb GEMMs on the 5th-gen tensor cores.
//
// Replaces kernels::dot_gr_ct_rows<16> / dot_prep_rows<16>
// (/root/reference/proj/src/kernels.cpp:29-53, include/irismpc/kernels.hpp:38-62):
// for every party p and dot d (code -> hd, mask -> ml)
//     C_p[row, col] = sum_k A_p[row, k] * B_p[col, k]   (mod 2^16)
// with 16-bit operands split into u8 limbs, V = lo + 256 hi:
//     C = A_lo.B_lo^T + 256 (A_lo.B_hi^T + A_hi.B_lo^T)   (mod 2^16)
// i.e. three tcgen05.mma.kind::i8 per k-step into two s32 TMEM accumulators
// (no saturation: the s32 wrap is harmless, only the low 16 bits survive).
// The epilogue recombines (acc0 + (acc1 << 8)) & 0xffff and writes the
// per-party additive shares in lane order (lane = col * s + row).
//
// Structure: one 128x256 output tile per CTA, warp-specialised:
//   warp 0   TMA producer (128B-swizzled K-major tiles, 2-stage mbarrier ring)
//   warp 1   single-thread tcgen05.mma issuer, tcgen05.commit -> mbarriers
//   warp 2   TMEM allocator (512 columns: acc0 | acc1)
//   warps 4-7 epilogue: tcgen05.ld -> recombine -> global stores
#include <cstdio>
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace irisgpu {

namespace {

constexpr int BM = kGemmBM, BN = kGemmBN, BK = kGemmBK;
constexpr int STAGES = 2;
constexpr int A_TILE = BM * BK;  // 16 KB
constexpr int B_TILE = BN * BK;  // 32 KB
constexpr int STAGE_BYTES = 2 * A_TILE + 2 * B_TILE;
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 256;
constexpr uint32_t TMEM_COLS = 512;

// UMMA shared-memory descriptor, K-major operand, 128B swizzle:
// start>>4 [0,14), LBO>>4 [16,30) (unused for SW128 K-major -> 1),
// SBO>>4 [32,46) = 1024 B between 8-row core groups, version 1 [46,48),
// layout SWIZZLE_128B = 2 at [61,64).
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// Instruction descriptor, kind::i8: c_format S32 (2) [4,6), a/b format u8 (0),
// K-major A and B, N>>3 [17,23), M>>4 [24,29).
constexpr uint32_t kIdesc = (2u << 4) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);

}  // namespace

__global__ void __launch_bounds__(256, 1)
    k_limb_gemm(const __grid_constant__ CUtensorMap tA_lo, const __grid_constant__ CUtensorMap tA_hi,
                const __grid_constant__ CUtensorMap tB_lo, const __grid_constant__ CUtensorMap tB_hi,
                const GemmArgs g) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* accum = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accum + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int n_tile = blockIdx.x;
  const int m_tile = blockIdx.y;
  const int prob = blockIdx.z;  // p * 2 + d
  const int p = prob >> 1, d = prob & 1;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tA_lo);
    tma_prefetch_desc(&tA_hi);
    tma_prefetch_desc(&tB_lo);
    tma_prefetch_desc(&tB_hi);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(accum, 1);
    fence_barrier_init();
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t nkb = g.nkb_seg * g.nseg;

  if (warp == 0) {
    if (lane == 0) {
      for (uint32_t kb = 0; kb < nkb; ++kb) {
        const uint32_t stage = kb % STAGES;
        const uint32_t phase = (kb / STAGES) & 1;
        mbar_wait(&empty[stage], phase ^ 1);
        const uint32_t seg = kb / g.nkb_seg;
        const uint32_t kk = kb % g.nkb_seg;
        const int pa = (g.rep && seg == 1) ? (p + 2) % 3 : p;  // A = [x_p | x_{p-1}]
        const int32_t arow = (int32_t)((uint32_t)(pa * 2 + d) * g.s_pad + g.row0 + m_tile * BM);
        const int32_t brow = (int32_t)(((uint32_t)prob * g.nseg + seg) * g.nb_rows + g.col0 + n_tile * BN);
        uint8_t* st = smem + stage * STAGE_BYTES;
        mbar_arrive_expect_tx(&full[stage], STAGE_BYTES);
        tma_load_2d(st, &tA_lo, &full[stage], (int32_t)(kk * BK), arow);
        tma_load_2d(st + A_TILE, &tA_hi, &full[stage], (int32_t)(kk * BK), arow);
        // B maps have a 128-row box (the CTA-pair kernel loads half tiles): two loads each
        tma_load_2d(st + 2 * A_TILE, &tB_lo, &full[stage], (int32_t)(kk * BK), brow);
        tma_load_2d(st + 2 * A_TILE + B_TILE / 2, &tB_lo, &full[stage], (int32_t)(kk * BK), brow + 128);
        tma_load_2d(st + 2 * A_TILE + B_TILE, &tB_hi, &full[stage], (int32_t)(kk * BK), brow);
        tma_load_2d(st + 2 * A_TILE + B_TILE + B_TILE / 2, &tB_hi, &full[stage], (int32_t)(kk * BK), brow + 128);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      for (uint32_t kb = 0; kb < nkb; ++kb) {
        const uint32_t stage = kb % STAGES;
        const uint32_t phase = (kb / STAGES) & 1;
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        const uint32_t st = smem_u32(smem + stage * STAGE_BYTES);
        const uint64_t dAlo = make_desc(st);
        const uint64_t dAhi = make_desc(st + A_TILE);
        const uint64_t dBlo = make_desc(st + 2 * A_TILE);
        const uint64_t dBhi = make_desc(st + 2 * A_TILE + B_TILE);
#pragma unroll
        for (int ks = 0; ks < BK / 32; ++ks) {
          const uint64_t off = (uint64_t)(ks * 32) >> 4;  // +32 bytes along K
          const uint32_t acc = (kb | ks) != 0;
          umma_i8(tmem, dAlo + off, dBlo + off, kIdesc, acc);            // lo.lo   -> acc0
          umma_i8(tmem + BN, dAlo + off, dBhi + off, kIdesc, acc);       // lo.hi   -> acc1
          umma_i8(tmem + BN, dAhi + off, dBlo + off, kIdesc, 1u);        // hi.lo   -> acc1
        }
        umma_commit(&empty[stage]);
      }
      umma_commit(accum);
    }
  } else if (warp >= 4) {
    mbar_wait(accum, 0);
    tc_fence_after();
    const int q = warp & 3;
    const uint32_t row = (uint32_t)m_tile * BM + q * 32 + lane;
    const uint32_t lane_addr = (uint32_t)(q * 32) << 16;
    uint16_t* out = g.out + (uint64_t)prob * g.out_pstride;
    const bool row_ok = row < g.s_valid;
#pragma unroll 1
    for (int c = 0; c < BN; c += 16) {
      uint32_t a0[16], a1[16];
      tmem_ld16(tmem + lane_addr + c, a0);
      tmem_ld16(tmem + lane_addr + BN + c, a1);
      tmem_wait_ld();
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const uint32_t col = (uint32_t)n_tile * BN + c + j;
        if (row_ok && col < g.ncols) {
          out[(uint64_t)col * g.out_cstride + row] = (uint16_t)((a0[j] + (a1[j] << 8)) & 0xFFFFu);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
  }
}

// ---------------------------------------------------------------- CTA pair
// cta_group::2 variant: a cluster of 2 CTAs computes a 256x256 tile; each CTA
// stages its own 128 DB rows and half (128 columns) of the query tile, the
// leader CTA issues tcgen05.mma.cta_group::2 (M = 256) and commits to both
// CTAs' barriers.  Per SM this halves the B traffic of the 1-CTA kernel
// (64 KB instead of 96 KB per 1536-cycle stage), which is what bounded it
// (L2 -> SM bandwidth, ncu: 69.8% tensor-pipe active).
namespace {
constexpr int P_STAGES = 3;
constexpr int PA_TILE = 128 * BK;  // 16 KB (this CTA's 128 rows)
constexpr int PB_TILE = 128 * BK;  // 16 KB (this CTA's 128 of 256 columns)
constexpr int P_STAGE = 2 * PA_TILE + 2 * PB_TILE;  // 64 KB
constexpr int P_SMEM = P_STAGES * P_STAGE + 1024 + 256;
constexpr uint32_t kIdescPair = (2u << 4) | ((uint32_t)(256 >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
}  // namespace

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 1)
    k_limb_gemm_pair(const __grid_constant__ CUtensorMap tA_lo, const __grid_constant__ CUtensorMap tA_hi,
                     const __grid_constant__ CUtensorMap tB_lo, const __grid_constant__ CUtensorMap tB_hi,
                     const GemmArgs g, uint32_t n_tiles, uint32_t m_pairs, uint32_t grouped) {
  // Persistent: clusters form groups of n_tiles; cluster c owns n_tile = c % n_tiles
  // and its group sweeps (prob, m_pair) units g, g + groups, ...  The n_tiles
  // clusters of a group read the same DB (A) k-blocks at the same time, so every
  // A byte comes from DRAM once; B (one problem's query tile, 26 MB) stays in L2.
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + P_STAGES * P_STAGE);
  uint64_t* empty = full + P_STAGES;
  uint64_t* accum = empty + P_STAGES;
  uint64_t* tmem_empty = accum + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const uint32_t ncl = gridDim.x >> 1;
  const uint32_t cl = blockIdx.x >> 1;
  // grouped: n_tiles clusters per group sweep the same (prob, m_pair) units;
  // flat (when grouping would idle SMs): a 1-cluster "group" walks tiles
  // t = cl, cl + ncl, ... over (unit, n_tile) with n_tile fastest.
  const bool flat = grouped == 0;
  const uint32_t tiles_per_unit = flat ? 1 : n_tiles;
  const uint32_t groups = ncl / tiles_per_unit;
  const uint32_t my_n = flat ? 0 : cl % n_tiles;
  const uint32_t g0 = flat ? cl : cl / n_tiles;
  const uint32_t nunits = flat ? 6 * m_pairs * n_tiles : 6 * m_pairs;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tA_lo);
    tma_prefetch_desc(&tA_hi);
    tma_prefetch_desc(&tB_lo);
    tma_prefetch_desc(&tB_hi);
    for (int s = 0; s < P_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(accum, 1);
    mbar_init(tmem_empty, 8);  // 4 epilogue warps x 2 CTAs
    fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t nkb = g.nkb_seg * g.nseg;

  if (warp == 0) {
    if (lane == 0) {
      uint32_t it = 0;
      for (uint32_t u = g0; u < nunits; u += groups) {
        const uint32_t n_tile = flat ? u % n_tiles : my_n;
        const uint32_t uu = flat ? u / n_tiles : u;
        const uint32_t m_pair = uu % m_pairs;
        const int prob = (int)(uu / m_pairs);
        const int p = prob >> 1, d = prob & 1;
        for (uint32_t kb = 0; kb < nkb; ++kb, ++it) {
          const uint32_t stage = it % P_STAGES;
          const uint32_t phase = (it / P_STAGES) & 1;
          mbar_wait(&empty[stage], phase ^ 1);
          const uint32_t seg = kb / g.nkb_seg;
          const uint32_t kk = kb % g.nkb_seg;
          const int pa = (g.rep && seg == 1) ? (p + 2) % 3 : p;  // A = [x_p | x_{p-1}]
          const int32_t arow = (int32_t)((uint32_t)(pa * 2 + d) * g.s_pad + g.row0 + m_pair * 256 + rank * 128);
          const int32_t brow =
              (int32_t)(((uint32_t)prob * g.nseg + seg) * g.nb_rows + g.col0 + n_tile * 256 + rank * 128);
          uint8_t* st = smem + stage * P_STAGE;
          if (leader) mbar_arrive_expect_tx(&full[stage], 2 * P_STAGE);
          const uint32_t fb = mapa_shared(&full[stage], 0);
          tma_load_2d_pair(st, &tA_lo, fb, (int32_t)(kk * BK), arow);
          tma_load_2d_pair(st + PA_TILE, &tA_hi, fb, (int32_t)(kk * BK), arow);
          tma_load_2d_pair(st + 2 * PA_TILE, &tB_lo, fb, (int32_t)(kk * BK), brow);
          tma_load_2d_pair(st + 2 * PA_TILE + PB_TILE, &tB_hi, fb, (int32_t)(kk * BK), brow);
        }
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {
      uint32_t it = 0, ti = 0;
      for (uint32_t u = g0; u < nunits; u += groups, ++ti) {
        if (ti > 0) {  // both CTAs' epilogues have drained the accumulators
          mbar_wait(tmem_empty, (ti - 1) & 1);
          tc_fence_after();
        }
        for (uint32_t kb = 0; kb < nkb; ++kb, ++it) {
          const uint32_t stage = it % P_STAGES;
          const uint32_t phase = (it / P_STAGES) & 1;
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t st = smem_u32(smem + stage * P_STAGE);
          const uint64_t dAlo = make_desc(st);
          const uint64_t dAhi = make_desc(st + PA_TILE);
          const uint64_t dBlo = make_desc(st + 2 * PA_TILE);
          const uint64_t dBhi = make_desc(st + 2 * PA_TILE + PB_TILE);
#pragma unroll
          for (int ks = 0; ks < BK / 32; ++ks) {
            const uint64_t off = (uint64_t)(ks * 32) >> 4;
            const uint32_t acc = (kb | ks) != 0;
            umma_i8_pair(tmem, dAlo + off, dBlo + off, kIdescPair, acc);        // lo.lo -> acc0
            umma_i8_pair(tmem + 256, dAlo + off, dBhi + off, kIdescPair, acc);  // lo.hi -> acc1
            umma_i8_pair(tmem + 256, dAhi + off, dBlo + off, kIdescPair, 1u);   // hi.lo -> acc1
          }
          umma_commit_pair(&empty[stage], 0x3);
        }
        umma_commit_pair(accum, 0x3);
      }
    }
  } else if (warp >= 4) {
    const int q = warp & 3;
    const uint32_t lane_addr = (uint32_t)(q * 32) << 16;
    const uint32_t te = mapa_shared(tmem_empty, 0);
    uint32_t ti = 0;
    for (uint32_t u = g0; u < nunits; u += groups, ++ti) {
      const uint32_t n_tile = flat ? u % n_tiles : my_n;
      const uint32_t uu = flat ? u / n_tiles : u;
      const uint32_t m_pair = uu % m_pairs;
      const int prob = (int)(uu / m_pairs);
      mbar_wait(accum, ti & 1);
      tc_fence_after();
      const uint32_t row = m_pair * 256 + rank * 128 + q * 32 + lane;
      uint16_t* out = g.out + (uint64_t)prob * g.out_pstride;
      const bool row_ok = row < g.s_valid;
#pragma unroll 1
      for (int c = 0; c < 256; c += 16) {
        uint32_t a0[16], a1[16];
        tmem_ld16(tmem + lane_addr + c, a0);
        tmem_ld16(tmem + lane_addr + 256 + c, a1);
        tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const uint32_t col = n_tile * 256 + c + j;
          if (row_ok && col < g.ncols)
            out[(uint64_t)col * g.out_cstride + row] = (uint16_t)((a0[j] + (a1[j] << 8)) & 0xFFFFu);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(te);
    }
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
  }
}

// ------------------------------------------------------------------ host

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                    const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                    const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled get_encode() {
  static PFN_encodeTiled fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled>(p);
  }
  return fn;
}

int make_plane_tmap(CUtensorMap* map, const void* base, uint64_t rows, uint64_t k_pad,
                    uint32_t box_rows) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return -1;
  const cuuint64_t dims[2] = {k_pad, rows};
  const cuuint64_t strides[1] = {k_pad};
  const cuuint32_t box[2] = {(cuuint32_t)BK, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box,
                   estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : (int)r;
}

void launch_gemm(const CUtensorMap& a_lo, const CUtensorMap& a_hi, const CUtensorMap& b_lo,
                 const CUtensorMap& b_hi, const GemmArgs& g, uint32_t m_tiles, uint32_t n_tiles,
                 cudaStream_t st) {
  static bool attr = false;
  static const bool one_cta = [] {
    const char* e = std::getenv("IRISMPC_GEMM_1CTA");  // A/B switch for the 1-CTA kernel
    return e && e[0] == '1';
  }();
  if (!attr) {
    cudaFuncSetAttribute(k_limb_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    cudaFuncSetAttribute(k_limb_gemm_pair, cudaFuncAttributeMaxDynamicSharedMemorySize, P_SMEM);
    attr = true;
  }
  if (one_cta) {
    dim3 grid(n_tiles, m_tiles, 6);
    k_limb_gemm<<<grid, 256, SMEM_BYTES, st>>>(a_lo, a_hi, b_lo, b_hi, g);
  } else {
    // m_tiles counts 128-row tiles; pairs cover 256 rows (s_pad is a multiple of 256).
    // Persistent: one CTA pair per two SMs.
    static int nsm = 0;
    if (!nsm) cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const uint32_t m_pairs = m_tiles / 2;
    const uint32_t units = 6 * m_pairs;
    const uint32_t max_cl = (uint32_t)(nsm / 2);
    const uint32_t groups = std::min<uint32_t>(units, max_cl / n_tiles);
    const bool grouped = groups >= 1 && (groups * n_tiles * 10 >= max_cl * 9 || groups == units);
    const uint32_t ncl = grouped ? groups * n_tiles : std::min<uint32_t>(units * n_tiles, max_cl);
    k_limb_gemm_pair<<<dim3(2 * ncl), 256, P_SMEM, st>>>(a_lo, a_hi, b_lo, b_hi, g, n_tiles, m_pairs,
                                                          grouped ? 1u : 0u);
  }
}

}  // namespace irisgpu
