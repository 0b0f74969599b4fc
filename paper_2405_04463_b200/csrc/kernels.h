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
// runtime switch (irismpc_gpu_profile) and read-out of the per-kernel totals (resets them)
void prof_enable(bool on);
size_t prof_take(char (*names)[48], double* ms, uint64_t* launches, size_t max);

// ---- variants (shares.hpp:28-48): ring widths of the hamming dot, the mask
// dot (0 = public mask bits) and the comparison
enum { kPlainMask = 0, kMpcLift = 1, kConstLift = 2, kNoLift = 3 };
struct VariantWidths {
  int kh, km, kc;
};
__host__ __device__ inline VariantWidths variant_widths(int v) {
  return {v == kNoLift ? 32 : 16, v == kPlainMask ? 0 : (v == kMpcLift ? 16 : 32), v == kPlainMask ? 16 : 32};
}

// One record field as stored in an IRS1 payload row (shares.hpp:52-56):
// `width` bytes per ring element (2 / 4) or 0 for l/8 public mask bytes.
struct FieldFmt {
  uint64_t rec_bytes;  // whole record (code + mask field)
  uint64_t off;        // byte offset of the field inside the record
  int width;           // 2, 4 or 0 (plain mask bits)
  int limbs;           // u8 limb planes of the field (width, or 1 for bits)
  int slot = -1;       // plane slot to write (-1: the party index)
  int take_prev = 0;   // replicated: keep the `prev` component instead of `own`
  int rp = 0;          // rotation-pair K layout (rp_pos), DB and query planes alike
};

// Rotation-pair (RP) K layout of an integer field's planes.  A plane row is
// H halves (Shamir: the lc0 | lc1 halves of l/2; replicated: one component of
// l) of 64 rotation blocks each (a rotation shifts a half by one block); the RP
// layout puts every half's even blocks first, then the odd ones:
//   row = [E_h0 .. E_h(H-1) | O_h0 .. O_h(H-1)],  E | O = l/2 elements each.
// A K-permutation applied to both GEMM operands leaves every dot unchanged;
// E and O (and S = E + O) are what the Winograd rotation-pair GEMM reads.
__host__ __device__ inline uint32_t rp_pos(uint32_t k, uint32_t l, int halves) {
  const uint32_t lh = l / halves, bs = lh / 64, h = k / lh, kk = k % lh, b = kk / bs, o = kk % bs;
  return (b & 1) * (l / 2) + h * (lh / 2) + (b >> 1) * bs + o;
}
// RP needs whole 4-element parse groups per block and l/2 a whole number of 128-byte k-blocks
inline bool rp_layout_ok(uint32_t l, int shamir) {
  const uint32_t bs = shamir ? l / 128 : l / 64;
  return l % 256 == 0 && bs % 4 == 0 && bs > 0;
}

// ---- K1 prep / dealer (prep.cu)
void set_lambda(const uint32_t lam[6]);
// DB-side planes of one field: planes[((c * limbs + limb) * s_pad + row0 + row) * l_pad + k]
// (c = party; bits: one public plane, c = 0)
void launch_parse_field(const uint8_t* pay, uint64_t nrows, uint64_t row0, uint32_t l, uint32_t l_pad,
                        uint64_t s_pad, int party, int shamir, const FieldFmt& f, uint8_t* planes,
                        cudaStream_t st);
void launch_check_rep(const uint8_t* p1, const uint8_t* p2, const uint8_t* p3, uint64_t nrows,
                      const FieldFmt& f, uint32_t l, int* bad, cudaStream_t st);
// Query-side rotated B planes of one field:
// planes[(((p * nseg + seg) * limbs + limb) * ncols_pad + col) * l_pad + k]
void launch_parse_query_field(const uint8_t* q1, const uint8_t* q2, const uint8_t* q3, uint32_t ncodes,
                              uint32_t l, uint32_t l_pad, uint32_t rot, uint32_t ncols_pad, int shamir,
                              const FieldFmt& f, uint8_t* planes, cudaStream_t st);
// RP: S = E + O (mod 2^(8 limbs)) of every DB plane row -> splanes[(c * limbs + limb) * s_pad + row][l / 2]
void launch_rp_sum(const uint8_t* planes, uint64_t ncomp, uint64_t s_pad, uint32_t l, uint32_t l_pad, int limbs,
                   uint8_t* splanes, cudaStream_t st);
// S = E + O for DB rows [row0, row0 + nrows) into a scratch of out_spad rows per plane
void launch_rp_sum_rows(const uint8_t* planes, uint64_t ncomp, uint64_t s_pad, uint64_t row0, uint64_t nrows,
                        uint64_t out_spad, uint32_t l, uint32_t l_pad, int limbs, uint8_t* splanes, cudaStream_t st);
// RP query planes: kinds D0 / M / D1 of the rotation pairs, rows
// [(((kind * 3 + p) * nseg + seg) * limbs + limb) * ncols_pad + code * npr + jp][l / 2]
void launch_parse_query_rp(const uint8_t* q1, const uint8_t* q2, const uint8_t* q3, uint32_t ncodes, uint32_t l,
                           uint32_t rot, uint32_t ncols_pad, int shamir, const FieldFmt& f, uint8_t* planes,
                           cudaStream_t st);
void launch_synth_records(SeedKey key, uint64_t first, uint64_t count, uint32_t l, double density,
                          uint64_t* codes, uint64_t* masks, cudaStream_t st);
void launch_deal(SeedKey key, uint64_t first_record, uint64_t nrec, uint32_t l, int shamir, int variant,
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
  uint32_t nseg;      // 1 (Shamir, public bits) or 2 (replicated [x_p | x_{p-1}])
  uint32_t rep;
  uint32_t nprob;     // 3 (one per party) or 1 (public mask popcount / one party's own dot)
  uint32_t limbs;     // 1 (0/1 bits), 2 (Z_2^16) or 4 (Z_2^32)
  uint32_t s_valid;   // rows written (relative to row0)
  uint32_t row0;      // first DB row of this launch (multiple of 256)
  uint32_t col0;      // first B row of this launch (chunk start column)
  uint32_t ncols;     // columns written (from col0)
  void* out;          // [nprob][ncols * out_cstride], u16 (limbs <= 2) or u32 (limbs = 4)
  uint64_t out_pstride;
  uint32_t out_cstride;
  uint32_t a_kb0 = 0;  // first A k-block of every segment (RP: the O half of a DB plane row)
  uint32_t b_row0 = 0; // B plane rows skipped (RP: the D0 / M / D1 plane set)
  // RP: one launch runs nkind = 3 products per party (problem = kind * nprob + party):
  // kind 0 P1 = E.D0 (A = tA), kind 1 P2 = S.M (A = tA2), kind 2 P3 = O.D1 (A = tA at a_kb0_k2)
  uint32_t nkind = 1;
  uint32_t a_kb0_k2 = 0;
  uint32_t b_kind_rows = 0;   // B rows per kind
  uint64_t out_kstride = 0;   // output elements per kind
  // kind-1 A rows (S planes) when they live in a per-chunk scratch: rows per plane and first row
  // (0 = the DB planes' s_pad / row0, resident S planes)
  uint32_t s_pad2 = 0;
  uint32_t row0_2 = 0;
  // kind-1 A operand S = E + O formed in shared memory from the E and O tiles of the
  // DB planes (no S planes in HBM): each kind-1 k-block takes two stage slots
  uint32_t s_conv = 0;
  // group lockstep (set by launch_gemm): per-cluster progress words, this launch's epoch
  unsigned long long* prog = nullptr;
  uint32_t epoch = 0;
  uint32_t lag = 16;  // k-block iterations a cluster may run ahead of its group's slowest
};
// N of one output tile: 256, or 128 for 4-limb operands (4 accumulators in 512 TMEM columns)
inline uint32_t gemm_bn(uint32_t limbs) { return limbs == 4 ? 128u : 256u; }
// Encodes the TMA map for a [rows][k_pad] u8 plane stack with a box of
// (128 bytes, box_rows) and 128B swizzle.  A maps use 128-row boxes; B maps
// gemm_bn(limbs) / 2 (each CTA of the pair stages half the tile's columns).
int make_plane_tmap(CUtensorMap* map, const void* base, uint64_t rows, uint64_t k_pad,
                    uint32_t box_rows);
void launch_gemm(const CUtensorMap& a, const CUtensorMap& b, const GemmArgs& g, uint32_t m_tiles,
                 uint32_t n_tiles, cudaStream_t st, const CUtensorMap* a2 = nullptr);
// cluster groups of the persistent GEMM: n_tiles clusters sweep one 256-row
// block of one problem in lockstep, groups of them run side by side
uint32_t gemm_groups(uint32_t n_tiles);

// ---- inner-batch pairs (pairs.cu)
// C: [nprob][ncols][ncodes] (elem_bytes each) -> out[p * out_pstride + pair lane]
void launch_pair_gather(const void* C, int elem_bytes, uint32_t nprob, uint32_t ncodes, uint32_t ncols,
                        uint32_t persons, uint32_t rot, void* out, uint64_t out_pstride, cudaStream_t st);

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
  int64_t slot;                   // partial slot of its first task (bucketed OR of sharded queries), -1 = none
  uint64_t src_rp;                // RP fields: chunk-buffer index of lane_begin in the P planes
  uint32_t rp_sel;                // RP fields: dot = P2 + P1 (1, odd rotation) or P2 + P3 (2, even)
};

struct ThrArgs {
  const Seg* segs;
  uint32_t nsegs;
  uint64_t ntasks, ngrp, ngblk;
  uint32_t ks_seg_threads;  // k_gate_keystream: max over the job's segments of 3 * ngates * blocks per row
  uint32_t grp_seg_max;     // max 8-lane groups of one segment (reshare / inject grid)
  uint32_t task_seg_max;    // max 1024-lane tasks of one segment (lift / msb grid)
  int variant;
  const void* hd[3];     // additive hd dots, u16 (KH = 16) or u32
  const void* ml[3];     // additive ml dots (u16 / u32), or the public popcount (u16, all three equal)
  // RP fields: hd / ml point at the party's P1 plane; P2, P3 follow at +rp_kstride, +2 rp_kstride
  // elements (0: the field's dots are plain [col][row])
  uint64_t rp_kstride_h, rp_kstride_m;
  uint64_t n, W;
  uint64_t pos[3];
  SeedKey key[3];
  uint32_t a, b;
  double coef;           // plain-mask: 1 - 2 * match_ratio (plain_threshold, iris.hpp:182-184)
  // AND-gate layout: gates [0, nlift) are the lift adder at lift_base[k] + g W,
  // gates [nlift, ngates) the MSB adder at msb_base[k] + (g - nlift) W
  uint32_t nlift, ngates;
  uint64_t lift_base[3], msb_base[3];
  uint64_t inj_base[3];  // bit_inject<15> draws of seeds 1 / 3 (mpc-lift): lift_base + 64 W
  int no_reshare;        // comparison-only (party_comparison_only): inputs are already replicated shares
  int tile_kernels;      // reshare / inject as 512-lane tiles (threshold.cu) instead of lane-major (threshold_lm.cu)
  // chunk work buffers
  uint64_t* gate;        // gate randomness, per segment [3*ngates][nwords]
  uint16_t* ml_rs;       // [3][cstride] reshared ml
  uint32_t* diff;        // [3][cstride] a*ml32 - b*hd
  uint64_t cstride;
  uint32_t* bits;        // [6][nbits] injected-bit rows (bit16 comps, bit17 comps)
  uint64_t nbits;
  uint32_t* match[3];    // optional 32-lane words (atomicOr), word = lane/32 - match_w0
  uint64_t match_w0;
  uint8_t* partial;      // [3][nslots]
  uint64_t nslots;
  uint64_t or_stream;    // ChaCha stream id of the fused OR gates (or_stream_id(ctr, rank, 1))
  uint64_t or_elem_base; // element base of this launch inside that stream
  // taps (tests), global-lane indexed, may be null
  uint32_t* tap_rs_hd;
  uint32_t* tap_rs_ml;
  uint32_t* tap_ml32;
  uint32_t* tap_diff;
  uint8_t* tap_msb;
};
// words of one (seed, gate) row of the gate buffer for a segment of nw reference
// words: nw / 8 + 2 whole ChaCha blocks (k_gate_keystream stores full blocks)
__host__ __device__ inline uint64_t gate_row_words(uint64_t nw) { return 8 * (nw / 8 + 2); }
void launch_threshold(const ThrArgs& a, cudaStream_t st);
// the chain in two halves for two streams: front = gate keystream + reshare (the
// dot readers), back = lift + inject + msb; parts: 1 front, 2 back, 3 both
void launch_threshold_front(const ThrArgs& a, cudaStream_t st);
void launch_threshold_back(const ThrArgs& a, cudaStream_t st);
void launch_threshold_part(const ThrArgs& a, cudaStream_t st, int parts);
// lane-major reshare / inject (threshold_lm.cu): the batch query's default (see launch_threshold)
void launch_reshare_lm(const ThrArgs& a, cudaStream_t st);
void launch_inject_lm(const ThrArgs& a, cudaStream_t st);
// comparison phase alone (party_comparison_only / party_or_tree_only, engine.cpp:448-532)
void launch_parse_lane_shares(const uint8_t* const p[3], uint64_t lanes, int width, void* out, int* bad,
                              cudaStream_t st);
void launch_parse_bit_shares(const uint8_t* const p[3], uint64_t words, uint64_t lanes, uint32_t* out, int* bad,
                             cudaStream_t st);
// L1 tap of an RP field's chunk: out[p * n + col * S + row0 + row] = P2 + P(1|3) of (col, row)
// row-sampled L1 tap (irismpc_gpu_tap_rows): out[p * out_pstride + col * k + i]
void launch_tap_rows(const void* P, int elem_bytes, uint32_t nparty, uint64_t ncols, uint32_t rot, uint64_t nr,
                     uint64_t kstride, const uint64_t* rows, uint32_t k, uint64_t row0, void* out,
                     uint64_t out_pstride, cudaStream_t st);
void launch_rp_tap(const void* P, int elem_bytes, uint32_t nparty, uint64_t ncols, uint32_t rot, uint64_t nr,
                   uint64_t kstride, void* out, uint64_t n, uint64_t S, uint64_t row0, cudaStream_t st);

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
  uint64_t stream;           // ChaCha stream id (or_stream_id(ctr, rank, 2)); person P uses elements P << 40 ...
  uint8_t* out;              // [3][persons] component bits
};
void launch_or_persons(const OrArgs& a, cudaStream_t st);
void launch_or_open(const uint8_t* partials, uint32_t G, uint32_t persons, const SeedKey key[3],
                    uint64_t stream, uint8_t* match_out, cudaStream_t st);

// Share-exact OR tree (ortree.cu): or_tree_batch over the reference's groups
struct OrTreeArgs {
  const uint64_t* match[3];  // lane bits in reference lane order, 64-lane words (+1 word of padding)
  uint32_t ngroups;          // persons, or 1 (membership / comparison: every lane)
  uint64_t db_lanes;         // group g's DB lanes: [g * db_lanes, (g + 1) * db_lanes)
  uint64_t pair_base;        // global lane of pair lane 0
  uint64_t pair_block;       // lanes per person pair (4 r), 0: no pair lanes
  uint64_t lanes;            // lanes per group = db_lanes + (ngroups - 1) * pair_block
  SeedKey key[3];
};
struct OrTreeLevel {
  uint64_t na, nb, wo, win;  // folded / AND lanes, out / in row strides (words)
  const uint64_t* in[3];
  uint64_t* out[3];
  uint64_t rand_base[3];     // stream element of group 0's first gate word, per seed
};
// u64 words of one ping-pong scratch buffer
uint64_t ortree_scratch_words(uint32_t ngroups, uint64_t lanes);
// all levels from the seed positions rand_start (the draws right after the msb
// gates), then lane 0 of every group -> out[3][ngroups]; returns launches
int launch_ortree(const OrTreeArgs& a, const uint64_t rand_start[3], uint64_t* scratch[2], uint8_t* out,
                  cudaStream_t st);

// ChaCha stream ids of the OR-reduction gates (the reference's own draws all use
// stream 0, prf.hpp:46-69): bit 63 set, a per-context 64-bit query counter
// (never reused on a persistent context), the shard rank and the kind
// (1 fused warp OR, 2 per-person OR, 3 cross-shard OR + open).  Every AND gate of
// every query therefore draws its zero shares from its own stream positions.
__host__ __device__ inline uint64_t or_stream_id(uint64_t ctr, uint32_t rank, uint32_t kind) {
  return (1ull << 63) | ((ctr & ((1ull << 43) - 1)) << 20) | ((uint64_t)(rank & 0xFFFFu) << 4) | (kind & 0xFu);
}
// element windows of k_or_persons: person P's linear items at P << 40, its block tree above 2^39
constexpr uint64_t kOrPersonShift = 40;
constexpr uint64_t kOrTreeOffset = 1ull << 39;

}  // namespace irisgpu
