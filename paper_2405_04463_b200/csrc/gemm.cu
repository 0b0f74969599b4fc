// K2: share dot products as u8-limb GEMMs on the 5th-gen tensor cores.
//
// Replaces kernels::dot_gr_ct_rows<K> / dot_prep_rows<K>
// (/root/reference/proj/src/kernels.cpp:29-61, include/irismpc/kernels.hpp:38-62)
// and the public-mask popcount_and (src/engine.cpp:62-68, 329-334): for every
// party p of one record field
//     C_p[row, col] = sum_k A_p[row, k] * B_p[col, k]   (mod 2^K)
// with the K-bit operands split into u8 limbs, V = sum_i 2^(8i) V_i:
//     C = sum_{i+j < L} 2^(8(i+j)) A_i.B_j^T            (mod 2^(8L))
// i.e. per k-step L(L+1)/2 tcgen05.mma.kind::i8 into L s32 TMEM accumulators
// (acc_s collects the products with i + j = s; the s32 wrap is harmless, only
// the low 8(L - s) bits of acc_s survive the recombination):
//     L = 1  public 0/1 mask bits: popcount(q & db) = acc0 (< 2^14)
//     L = 2  Z_2^16: 3 MMAs, 2 accumulators, N = 256
//     L = 4  Z_2^32: 10 MMAs, 4 accumulators, N = 128 (4 x 128 TMEM columns)
// The epilogue recombines sum_s acc_s << 8s and writes the per-party additive
// shares in lane order (lane = col * s + row).
//
// cta_group::2: a cluster of 2 CTAs computes a 256 x N tile; each CTA stages
// its own 128 DB rows and N/2 query columns per limb, the leader CTA issues
// tcgen05.mma.cta_group::2 (M = 256) and commits to both CTAs' barriers.
// Warp-specialised and persistent:
//   warp 0   TMA producer (128B-swizzled K-major tiles, mbarrier ring)
//   warp 1   TMEM allocator; the leader's lane 0 issues the MMAs
//   warps 2-9 epilogue: tcgen05.ld -> recombine -> global stores; two warps per
//            TMEM lane quadrant, each draining half of the tile's columns
// (10 warps: the accumulators of a 256 x 256 tile fill all 512 TMEM columns, so
// the epilogue is exposed once per tile; 8 warps drain it in half the time of 4
// (-2% GEMM, -1% query), 16 crowd out the threshold kernels that run
// concurrently on the second stream (+8% query))
#include <cstdio>
#include <algorithm>
#include <cstdlib>
#include <atomic>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "kernels.h"

namespace irisgpu {

namespace {

constexpr int BK = kGemmBK;
// epilogue warps (multiple of 4: one per TMEM lane quadrant per column slice)
#ifndef GEMM_EPI_WARPS
#define GEMM_EPI_WARPS 8
#endif
constexpr int kEpiWarps = GEMM_EPI_WARPS;
constexpr int kGemmThreads = 32 * (2 + kEpiWarps);
constexpr uint32_t TMEM_COLS = 512;
constexpr int kStageBudget = 200 * 1024;

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

template <int L>
struct Tile {
  static constexpr int BN = L == 4 ? 128 : 256;       // output columns per tile
  static constexpr int A_T = 128 * BK;                // this CTA's 128 rows, one limb
  static constexpr int B_T = (BN / 2) * BK;           // this CTA's BN/2 columns, one limb
  static constexpr int STAGE = L * (A_T + B_T);
  static constexpr int STAGES = kStageBudget / STAGE > 6 ? 6 : kStageBudget / STAGE;
  static constexpr int SMEM = STAGES * STAGE + 1024 + 256;
  // Instruction descriptor, kind::i8: c_format S32 (2) [4,6), a/b format u8 (0),
  // K-major A and B, N>>3 [17,23), M>>4 [24,29) with M = 256 (CTA pair).
  static constexpr uint32_t IDESC = (2u << 4) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
};

}  // namespace

template <int L, bool CONV>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kGemmThreads, 1)
    k_limb_gemm_pair(const __grid_constant__ CUtensorMap tA, const __grid_constant__ CUtensorMap tB,
                     const __grid_constant__ CUtensorMap tA2,
                     const GemmArgs g, uint32_t n_tiles, uint32_t m_pairs, uint32_t grouped) {
  // Persistent: clusters form groups of n_tiles; cluster c owns n_tile = c % n_tiles
  // and its group sweeps (prob, m_pair) units g, g + groups, ...  The n_tiles
  // clusters of a group read the same DB (A) k-blocks at the same time, so every
  // A byte comes from DRAM once; B (one problem's query tile) stays in L2.
  using T = Tile<L>;
  constexpr int BN = T::BN, STAGES = T::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * T::STAGE);
  uint64_t* empty = full + STAGES;
  uint64_t* accum = empty + STAGES;
  uint64_t* tmem_empty = accum + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 1);
  // s_conv: raw[s] = this CTA's E / O tile landed in slot s (local TMA), conv[s] (leader) =
  // both CTAs' epilogue warps have written S into slot s
  uint64_t* raw = reinterpret_cast<uint64_t*>(smem + STAGES * T::STAGE + 128);
  uint64_t* conv = raw + STAGES;

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
  const uint32_t nprob_all = g.nprob * g.nkind;
  const uint32_t nunits = flat ? nprob_all * m_pairs * n_tiles : nprob_all * m_pairs;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tA);
    if (g.nkind > 1) tma_prefetch_desc(&tA2);
    tma_prefetch_desc(&tB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(accum, 1);
    mbar_init(tmem_empty, 2 * kEpiWarps);  // epilogue warps x 2 CTAs
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&raw[s], 1);
      mbar_init(&conv[s], 2 * kEpiWarps);
    }
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
    // TMA producer: warp-uniform loop, one elected lane issues.
    // Group lockstep: the n_tiles clusters of a group read the same A k-blocks; left
    // alone they drift apart by more than the L2 holds and each re-reads A from DRAM
    // (3.3x the DB planes at configs[2]).  The leader CTA of each cluster publishes
    // the k-block iteration it has issued and does not run more than kLag
    // iterations ahead of the slowest cluster of its group (a bounded wait: the
    // progress words are only a scheduling hint, never a correctness condition).
    const uint32_t kLag = g.lag;
    bool lock = !flat && n_tiles > 1 && n_tiles <= 32 && g.prog != nullptr && leader;
    const uint32_t grp_base = (cl / tiles_per_unit) * tiles_per_unit;
    uint32_t seen = 0;
    uint32_t it = 0;
    for (uint32_t u = g0; u < nunits; u += groups) {
      const uint32_t n_tile = flat ? u % n_tiles : my_n;
      const uint32_t uu = flat ? u / n_tiles : u;
      const uint32_t m_pair = uu % m_pairs;
      const uint32_t prob = uu / m_pairs;
      const uint32_t kind = prob / g.nprob, p = prob % g.nprob;
      const void* ta = kind == 1 ? (const void*)&tA2 : (const void*)&tA;
      const uint32_t akb = kind == 2 ? g.a_kb0_k2 : g.a_kb0;
      const bool s_scratch = kind == 1 && g.s_pad2 != 0;  // per-chunk S planes
      const uint32_t a_spad = s_scratch ? g.s_pad2 : g.s_pad, a_row0 = s_scratch ? g.row0_2 : g.row0;
      const uint32_t brow0 = g.b_row0 + kind * g.b_kind_rows;
      const bool cv = CONV && kind == 1;
      for (uint32_t kb = 0; kb < nkb; ++kb, ++it) {
        const uint32_t stage = it % STAGES;
        const uint32_t phase = (it / STAGES) & 1;
        if constexpr (CONV) if (cv) {
          // E tiles into slot s0's A part, O tiles into slot s1's A part (local TMA, this
          // CTA's raw barriers), B into slot s0 (pair TMA, leader's full barrier); the
          // epilogue warps add them into S in place (slot s0), the MMA reads slot s0
          const uint32_t s1 = (it + 1) % STAGES, ph1 = ((it + 1) / STAGES) & 1;
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_wait(&empty[s1], ph1 ^ 1);
          const uint32_t seg = kb / g.nkb_seg, kk = kb % g.nkb_seg;
          const uint32_t pa = (g.rep && seg == 1) ? (p + 2) % 3 : p;
          uint8_t* st0 = smem + stage * T::STAGE;
          uint8_t* st1 = smem + s1 * T::STAGE;
          if (elect_one()) {
            if (leader) {
              mbar_arrive_expect_tx(&full[stage], 2 * L * T::B_T);
              mbar_arrive_expect_tx(&full[s1], 0);
            }
            mbar_arrive_expect_tx(&raw[stage], L * T::A_T);
            mbar_arrive_expect_tx(&raw[s1], L * T::A_T);
            const uint32_t fb = mapa_shared(&full[stage], 0);
#pragma unroll
            for (int limb = 0; limb < L; ++limb) {
              const int32_t arow = (int32_t)((pa * L + limb) * g.s_pad + g.row0 + m_pair * 256 + rank * 128);
              const int32_t brow = (int32_t)(brow0 + ((p * g.nseg + seg) * L + limb) * g.nb_rows + g.col0 +
                                             n_tile * BN + rank * (BN / 2));
              tma_load_2d(st0 + limb * T::A_T, &tA, &raw[stage], (int32_t)((g.a_kb0 + kk) * BK), arow);
              tma_load_2d(st1 + limb * T::A_T, &tA, &raw[s1], (int32_t)((g.a_kb0_k2 + kk) * BK), arow);
              tma_load_2d_pair(st0 + L * T::A_T + limb * T::B_T, &tB, fb, (int32_t)(kk * BK), brow);
            }
            if (lock) {
              const unsigned long long w = ((unsigned long long)g.epoch << 32) | (it + 2);
              asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(g.prog + cl), "l"(w) : "memory");
            }
          }
          __syncwarp();
          ++it;  // the second slot
          continue;
        }
        if (lock && it >= kLag + seen) {
          uint64_t t0;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
          for (;;) {
            uint32_t v = 0xFFFFFFFFu;
            if ((uint32_t)lane < n_tiles) {
              unsigned long long w;
              asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(w) : "l"(g.prog + grp_base + lane));
              v = (uint32_t)(w >> 32) == g.epoch ? (uint32_t)w : 0u;
            }
            v = __reduce_min_sync(0xFFFFFFFFu, v);
            seen = v;
            if (it < kLag + v) break;
            uint64_t t1;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
            if (t1 - t0 > 50000) {  // a group member is not running (not yet resident): stop pacing
              lock = false;
              break;
            }
            __nanosleep(128);
          }
        }
        mbar_wait(&empty[stage], phase ^ 1);
        const uint32_t seg = kb / g.nkb_seg;
        const uint32_t kk = kb % g.nkb_seg;
        // A = [x_p | x_{p-1}]: the previous party's component plane, or plane 1
        // of a single party's (own, prev) planes (party mode, nprob = 1)
        const uint32_t pa = (g.rep && seg == 1) ? (g.nprob == 1 ? 1u : (p + 2) % 3) : p;
        uint8_t* st = smem + stage * T::STAGE;
        if (elect_one()) {
          if (leader) mbar_arrive_expect_tx(&full[stage], 2 * T::STAGE);
          const uint32_t fb = mapa_shared(&full[stage], 0);
#pragma unroll
          for (int limb = 0; limb < L; ++limb) {
            const int32_t arow = (int32_t)((pa * L + limb) * a_spad + a_row0 + m_pair * 256 + rank * 128);
            const int32_t brow = (int32_t)(brow0 + ((p * g.nseg + seg) * L + limb) * g.nb_rows + g.col0 +
                                           n_tile * BN + rank * (BN / 2));
            tma_load_2d_pair(st + limb * T::A_T, ta, fb, (int32_t)((akb + kk) * BK), arow);
            tma_load_2d_pair(st + L * T::A_T + limb * T::B_T, &tB, fb, (int32_t)(kk * BK), brow);
          }
          if (lock) {
            const unsigned long long w = ((unsigned long long)g.epoch << 32) | (it + 1);
            asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(g.prog + cl), "l"(w) : "memory");
          }
        }
        __syncwarp();
      }
    }
  } else if (warp == 1) {
    // MMA issuer (leader CTA): warp-uniform loop, one elected lane issues
    if (leader) {
      uint32_t it = 0, ti = 0, convph = 0;
      for (uint32_t u = g0; u < nunits; u += groups, ++ti) {
        if (ti > 0) {  // both CTAs' epilogues have drained the accumulators
          mbar_wait(tmem_empty, (ti - 1) & 1);
          tc_fence_after();
        }
        const uint32_t uu = flat ? u / n_tiles : u;
        const bool cv = CONV && (uu / m_pairs) / g.nprob == 1;
        for (uint32_t kb = 0; kb < nkb; ++kb, ++it) {
          const uint32_t stage = it % STAGES;
          const uint32_t phase = (it / STAGES) & 1;
          mbar_wait(&full[stage], phase);
          uint32_t s1 = 0;
          if (cv) {  // B landed (full) and both CTAs' S tiles written (conv); slot s1 is released with s0
            s1 = (it + 1) % STAGES;
            mbar_wait(&conv[stage], (convph >> stage) & 1);
            convph ^= 1u << stage;
          }
          tc_fence_after();
          const uint32_t st = smem_u32(smem + stage * T::STAGE);
          if (elect_one()) {
#pragma unroll
            for (int ks = 0; ks < BK / 32; ++ks) {
              const uint64_t off = (uint64_t)(ks * 32) >> 4;  // +32 bytes along K
#pragma unroll
              for (int i = 0; i < L; ++i)
#pragma unroll
                for (int j = 0; i + j < L; ++j) {
                  const uint64_t da = make_desc(st + i * T::A_T) + off;
                  const uint64_t db = make_desc(st + L * T::A_T + j * T::B_T) + off;
                  const uint32_t acc = ((kb | ks) != 0 || i > 0) ? 1u : 0u;  // (0, s) opens acc_s
                  umma_i8_pair(tmem + (i + j) * BN, da, db, T::IDESC, acc);
                }
            }
            umma_commit_pair(&empty[stage], 0x3);
            if (cv) umma_commit_pair(&empty[s1], 0x3);
          }
          __syncwarp();
          if (cv) ++it;
        }
        if (elect_one()) umma_commit_pair(accum, 0x3);
        __syncwarp();
      }
    }
  } else if (warp >= 2) {
    const int q = warp & 3;  // tcgen05.ld: warp w reads TMEM lanes 32 (w % 4) .. + 31
    // kEpiWarps / 4 warps share a lane quadrant, each draining its slice of the columns
    constexpr int kSlice = BN / (kEpiWarps / 4);
    const int c0 = ((warp - 2) / 4) * kSlice;
    const uint32_t lane_addr = (uint32_t)(q * 32) << 16;
    const uint32_t te = mapa_shared(tmem_empty, 0);
    uint32_t ti = 0, cit = 0, rawph = 0;
    const int et = threadIdx.x - 64;  // 0 .. 32 kEpiWarps - 1
    for (uint32_t u = g0; u < nunits; u += groups, ++ti) {
      const uint32_t n_tile = flat ? u % n_tiles : my_n;
      const uint32_t uu = flat ? u / n_tiles : u;
      const uint32_t m_pair = uu % m_pairs;
      const uint32_t prob = uu / m_pairs;
      const uint32_t kind = prob / g.nprob, p = prob % g.nprob;
      if (CONV && kind == 1) {
        // S = E + O (mod 2^(8L), limb-wise with carries) in place in slot s0's A tiles; both
        // tiles carry the same 128B swizzle, so equal byte offsets hold the same (row, k)
        for (uint32_t kb = 0; kb < nkb; ++kb, cit += 2) {
          const uint32_t s0 = cit % STAGES, s1 = (cit + 1) % STAGES;
          mbar_wait(&raw[s0], (rawph >> s0) & 1);
          rawph ^= 1u << s0;
          mbar_wait(&raw[s1], (rawph >> s1) & 1);
          rawph ^= 1u << s1;
          uint4* e = reinterpret_cast<uint4*>(smem + s0 * T::STAGE);
          const uint4* o = reinterpret_cast<const uint4*>(smem + s1 * T::STAGE);
          constexpr int kVec = T::A_T / 16;  // uint4 per limb tile
#pragma unroll 2
          for (int v = et; v < kVec; v += 32 * kEpiWarps) {
            uint32_t c[4] = {0u, 0u, 0u, 0u};
#pragma unroll
            for (int limb = 0; limb < L; ++limb) {
              const uint4 a = e[limb * kVec + v], b = o[limb * kVec + v];
              const uint32_t x[4] = {a.x, a.y, a.z, a.w}, y[4] = {b.x, b.y, b.z, b.w};
              uint32_t r[4];
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const uint32_t t = __vadd4(x[i], y[i]);
                r[i] = __vadd4(t, c[i]);
                if (limb + 1 < L) {
                  const uint32_t c1 = ((x[i] & y[i]) | ((x[i] | y[i]) & ~t)) & 0x80808080u;
                  const uint32_t c2 = t & ~r[i] & 0x80808080u;
                  c[i] = (c1 | c2) >> 7;
                }
              }
              e[limb * kVec + v] = make_uint4(r[0], r[1], r[2], r[3]);
            }
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(mapa_shared(&conv[s0], 0));
        }
      } else {
        cit += nkb;
      }
      mbar_wait(accum, ti & 1);
      tc_fence_after();
      const uint32_t row = m_pair * 256 + rank * 128 + q * 32 + lane;
      const bool row_ok = row < g.s_valid;
#pragma unroll 1
      for (int c = c0; c < c0 + kSlice; c += 16) {
        uint32_t acc[L][16];
#pragma unroll
        for (int s = 0; s < L; ++s) tmem_ld16(tmem + lane_addr + s * BN + c, acc[s]);
        tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const uint32_t col = n_tile * BN + c + j;
          if (!row_ok || col >= g.ncols) continue;
          uint32_t v = acc[0][j];
#pragma unroll
          for (int s = 1; s < L; ++s) v += acc[s][j] << (8 * s);
          const uint64_t o = kind * g.out_kstride + (uint64_t)p * g.out_pstride + (uint64_t)col * g.out_cstride + row;
          if (L == 4)
            static_cast<uint32_t*>(g.out)[o] = v;
          else
            static_cast<uint16_t*>(g.out)[o] = (uint16_t)v;
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

// Per-device launch state: the >48 KB dynamic shared-memory opt-in is a
// per-device function attribute and the SM count differs per device, so both
// are kept per CUDA device ordinal (a process may hold contexts on several
// GPUs, and party threads launch concurrently).
namespace {
constexpr int kMaxDev = 64;
struct DevState {
  std::once_flag attr[6];  // dynamic-smem opt-in of k_limb_gemm_pair<1 / 2 / 4, CONV>
  std::once_flag sms;
  int nsm = 0;
  // group-lockstep progress words (one per cluster), one buffer per stream: GEMMs of
  // different streams (contexts) may run concurrently
  std::mutex prog_mu;
  std::vector<std::pair<cudaStream_t, unsigned long long*>> prog;
  std::atomic<uint32_t> epoch{0};
};
DevState g_dev[kMaxDev];

int cur_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d < 0 ? 0 : (d >= kMaxDev ? kMaxDev - 1 : d);
}

int device_sms(int d) {
  DevState& s = g_dev[d];
  std::call_once(s.sms, [&] {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d);
    if (const char* e = std::getenv("IRISMPC_GEMM_SMS")) n = std::max(2, std::min(n, std::atoi(e)));  // experiment hook
    s.nsm = n;
  });
  return s.nsm;
}
}  // namespace

template <int L, bool CONV>
static void launch_pair_kernel(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& a2, const GemmArgs& g,
                               uint32_t m_tiles, uint32_t n_tiles, cudaStream_t st) {
  using T = Tile<L>;
  const int dev = cur_device();
  constexpr int slot = (L == 1 ? 0 : (L == 2 ? 1 : 2)) + (CONV ? 3 : 0);
  std::call_once(g_dev[dev].attr[slot], [] {
    cudaFuncSetAttribute(k_limb_gemm_pair<L, CONV>, cudaFuncAttributeMaxDynamicSharedMemorySize, T::SMEM);
  });
  // m_tiles counts 128-row tiles; pairs cover 256 rows (s_pad is a multiple of 256).
  // Persistent: one CTA pair per two SMs.
  const int nsm = device_sms(dev);
  const uint32_t m_pairs = m_tiles / 2;
  const uint32_t units = g.nprob * g.nkind * m_pairs;
  const uint32_t max_cl = (uint32_t)(nsm / 2);
  const uint32_t groups = std::min<uint32_t>(units, max_cl / n_tiles);
  const bool grouped = groups >= 1 && (groups * n_tiles * 10 >= max_cl * 9 || groups == units);
  const uint32_t ncl = grouped ? groups * n_tiles : std::min<uint32_t>(units * n_tiles, max_cl);
  GemmArgs ga = g;
  static const bool no_lock = std::getenv("IRISMPC_GEMM_NO_LOCKSTEP") != nullptr;  // A/B hook
  if (grouped && n_tiles > 1 && !no_lock) {
    DevState& ds = g_dev[dev];
    unsigned long long* pg = nullptr;
    {
      std::lock_guard<std::mutex> lk(ds.prog_mu);
      for (auto& e : ds.prog)
        if (e.first == st) pg = e.second;
      if (!pg && cudaMalloc(&pg, 1024 * sizeof(unsigned long long)) == cudaSuccess) {
        cudaMemset(pg, 0, 1024 * sizeof(unsigned long long));
        ds.prog.emplace_back(st, pg);
      } else if (!pg) {
        cudaGetLastError();
      }
    }
    if (pg && ncl <= 1024) {
      ga.prog = pg;
      static const uint32_t lag = [] {
        const char* e = std::getenv("IRISMPC_GEMM_LAG");  // A/B hook
        return e ? (uint32_t)std::max(1, std::atoi(e)) : 16u;
      }();
      ga.lag = lag;
      ga.epoch = ++ds.epoch;  // launches on one device are ordered per stream; epochs tell them apart
      if (ga.epoch == 0) ga.epoch = ++ds.epoch;
    }
  }
  k_limb_gemm_pair<L, CONV><<<dim3(2 * ncl), kGemmThreads, T::SMEM, st>>>(a, b, a2, ga, n_tiles, m_pairs,
                                                                         grouped ? 1u : 0u);
}

uint32_t gemm_groups(uint32_t n_tiles) {
  const int nsm = device_sms(cur_device());
  return std::max<uint32_t>(1, (uint32_t)(nsm / 2) / std::max<uint32_t>(1, n_tiles));
}

void launch_gemm(const CUtensorMap& a, const CUtensorMap& b, const GemmArgs& g, uint32_t m_tiles,
                 uint32_t n_tiles, cudaStream_t st, const CUtensorMap* a2) {
  const CUtensorMap& A2 = a2 ? *a2 : a;
  switch (g.limbs) {
    case 1: launch_pair_kernel<1, false>(a, b, A2, g, m_tiles, n_tiles, st); break;
    case 2:
      if (g.s_conv)
        launch_pair_kernel<2, true>(a, b, A2, g, m_tiles, n_tiles, st);
      else
        launch_pair_kernel<2, false>(a, b, A2, g, m_tiles, n_tiles, st);
      break;
    default:
      if (g.s_conv)
        launch_pair_kernel<4, true>(a, b, A2, g, m_tiles, n_tiles, st);
      else
        launch_pair_kernel<4, false>(a, b, A2, g, m_tiles, n_tiles, st);
      break;
  }
}

}  // namespace irisgpu
