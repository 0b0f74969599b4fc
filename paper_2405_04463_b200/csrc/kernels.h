// Internal launcher declarations shared by the .cu files and the C-ABI layer.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"

namespace irisgpu {

// IRISMPC_DEBUG_SYNC=1: synchronize after every launch and abort with the
// kernel's name on a device fault (no sanitizer on this pool).
void debug_check(const char* what, cudaStream_t st);
// IRISMPC_PROFILE=1: bracket launches with CUDA events (per-kernel totals at exit)
bool prof_on();
void* prof_begin(cudaStream_t st);
void prof_end(void* h, const char* name, cudaStream_t st);

// ---- K1 prep / dealer (prep.cu)
void set_lambda(const uint16_t lam[6]);
void launch_parse_db(const uint8_t* pay, uint64_t nrows, uint64_t row0, uint32_t l, uint32_t l_pad,
                     uint64_t s_pad, int party, int shamir, uint8_t* lo, uint8_t* hi,
                     cudaStream_t st);
void launch_check_rep(const uint8_t* p1, const uint8_t* p2, const uint8_t* p3, uint64_t bytes,
                      int* bad, cudaStream_t st);
void launch_parse_query(const uint8_t* q1, const uint8_t* q2, const uint8_t* q3, uint32_t ncodes,
                        uint32_t l, uint32_t l_pad, uint32_t rot, uint32_t ncols_pad, int shamir,
                        uint8_t* blo, uint8_t* bhi, uint16_t* pa, uint16_t* pb, cudaStream_t st);
void launch_synth_records(SeedKey key, uint64_t first, uint64_t count, uint32_t l, double density,
                          uint64_t* codes, uint64_t* masks, cudaStream_t st);
void launch_deal(SeedKey key, uint64_t first_record, uint64_t nrec, uint32_t l, int shamir,
                 const uint64_t* codes, const uint64_t* masks, uint8_t* o1, uint8_t* o2,
                 uint8_t* o3, cudaStream_t st);

// ---- K2 limb GEMM (gemm.cu)
constexpr int kGemmBM = 128;
constexpr int kGemmBN = 256;
constexpr int kGemmBK = 128;

struct GemmArgs {
  uint32_t s_pad;     // rows per A plane
  uint32_t nb_rows;   // rows per B plane (ncols_pad)
  uint32_t nkb_seg;   // k-blocks per K segment (l_pad / 128)
  uint32_t nseg;      // 1 (Shamir) or 2 (replicated [x_p | x_{p-1}])
  uint32_t rep;
  uint32_t s_valid;   // rows written (relative to row0)
  uint32_t row0;      // first DB row of this launch (multiple of 256)
  uint32_t col0;      // first B row of this launch (chunk start column)
  uint32_t ncols;     // columns written (from col0)
  uint16_t* out;      // [6][ncols * out_cstride]
  uint64_t out_pstride;
  uint32_t out_cstride;
};
// Encodes the TMA map for a [rows][k_pad] u8 plane stack with a box of
// (128 bytes, box_rows) and 128B swizzle.
int make_plane_tmap(CUtensorMap* map, const void* base, uint64_t rows, uint64_t k_pad,
                    uint32_t box_rows);
void launch_gemm(const CUtensorMap& a_lo, const CUtensorMap& a_hi, const CUtensorMap& b_lo,
                 const CUtensorMap& b_hi, const GemmArgs& g, uint32_t m_tiles, uint32_t n_tiles,
                 cudaStream_t st);

// ---- inner-batch pairs (pairs.cu)
void launch_pair_gather(const uint16_t* C, uint32_t ncodes, uint32_t ncols, uint32_t persons, uint32_t rot,
                        uint16_t* out_hd, uint16_t* out_ml, uint64_t out_pstride, cudaStream_t st);

// ---- K4 threshold (threshold.cu)
struct Seg {
  uint64_t lane_begin, lane_end;  // global lanes [begin, end)
  uint64_t src;                   // chunk-buffer index of lane_begin
  uint64_t task_begin;            // first 1024-lane task of this segment (chunk-relative)
  uint64_t q_first;               // lane_begin / 1024
  uint64_t w_first;               // lane_begin / 64 (first reference word)
  uint64_t g_off;                 // u64 offset of this segment's gate randomness block
  uint64_t grp_begin;             // first 8-lane group (chunk-relative)
  uint64_t gblk_begin;            // first gate-keystream thread (chunk-relative)
  int64_t slot;                   // partial slot of its first task, -1 = no fused OR
};

struct ThrArgs {
  const Seg* segs;
  uint32_t nsegs;
  uint64_t ntasks, ngrp, ngblk;
  const uint16_t* hd[3];
  const uint16_t* ml[3];
  uint64_t n, W;
  uint64_t pos[3];
  SeedKey key[3];
  uint32_t a, b;
  // chunk work buffers
  uint64_t* gate;        // gate randomness, per segment [3*125][nwords]
  uint16_t* ml_rs;       // [3][cstride] reshared ml
  uint32_t* diff;        // [3][cstride] a*ml32 - b*hd
  uint64_t cstride;
  uint32_t* bits;        // [6][nbits] injected-bit rows (bit16 comps, bit17 comps)
  uint64_t nbits;
  uint32_t* match[3];    // optional 32-lane words (atomicOr), word = lane/32 - match_w0
  uint64_t match_w0;
  uint8_t* partial;      // [3][nslots]
  uint64_t nslots;
  uint64_t or_elem_base; // OR-stream (stream id 1) element base of this launch
  // taps (tests), global-lane indexed, may be null
  uint16_t* tap_rs_hd;
  uint16_t* tap_rs_ml;
  uint32_t* tap_ml32;
  uint32_t* tap_diff;
  uint8_t* tap_msb;
};
void launch_threshold(const ThrArgs& a, cudaStream_t st);

// ---- K5 OR reduction + open (orreduce.cu)
struct OrArgs {
  const uint8_t* partial;   // [3][nslots]
  uint64_t nslots;
  const uint64_t* slot_begin;  // [persons + 1] per-person slot ranges (device)
  const uint32_t* pair_match[3];  // pair lane bits (words), may be null
  uint64_t pair_w0;          // word index of pair lane 0's word
  uint64_t pair_lane0;       // global lane of pair lane 0
  uint32_t persons, rot;
  SeedKey key[3];
  uint64_t elem_base;        // OR stream (stream id 2) element base
  uint8_t* out;              // [3][persons] component bits
};
void launch_or_persons(const OrArgs& a, cudaStream_t st);
void launch_or_open(const uint8_t* partials, uint32_t G, uint32_t persons, const SeedKey key[3],
                    uint64_t elem_base, uint8_t* match_out, cudaStream_t st);

}  // namespace irisgpu
