// f3: the query with ONE PARTY per process / GPU (the reference's deployment,
// PAPER.md:508-512), all four variants.  Each party holds only its own IRS1 payloads
// and its two seeds (own = seed_p, prev = seed_{p-1}); every protocol message
// of the reference crosses a real transport, round by round:
//
//   dot      reshare_pair<KH,KM>: own -> next party                (engine.cpp:80-106)
//   lift     (mpc-lift) bit_extract_sum {16,17}: 1 FA + 16 chain rounds (circuits.hpp:202-296)
//   ot       (mpc-lift) bit_inject<15>, <16>: P1 -> P2, P3 -> P2, then P2 -> P3 (convert.hpp:42-155)
//   msb      msb_batch<KC>: 1 FA round + KC - 2 chain rounds
//   or_tree  [debug_rows open], or_tree_batch halving rounds, open_bits_to(P1)
//            (circuits.hpp:387-486)
//
// Transports: NCCL send/recv (ranks 0,1,2 = parties 1,2,3; libnccl loaded at
// run time so the library has no link-time NCCL dependency) or an in-process
// mailbox for three party contexts in one process (InProcNet analogue,
// transport.hpp:129-154).  The ledger counts what the reference's CommLedger
// counts (bytes per phase as the reference serialises them, rounds per phase).
//
// Every share equals the reference's (component p and p-1 of the
// component-form simulation): the PRF draws use the same stream indices as
// the single-GPU engine, and the OR tree is the reference's
// halving tree, so even the aggregate shares and the stream positions match.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/irismpc_gpu.h"
#include "common.cuh"
#include "kernels.h"
#include "nccl_api.h"

using namespace irisgpu;

namespace {

constexpr int kThreads = 256;
// at least one block: a query with zero lanes still runs every protocol round
// (empty messages, the reference's ledger); every kernel bounds-checks
inline unsigned nblk(uint64_t n, unsigned b = kThreads) { return n ? (unsigned)((n + b - 1) / b) : 1u; }
__host__ __device__ inline uint64_t cdiv(uint64_t a, uint64_t b) { return (a + b - 1) / b; }
inline uint64_t rup(uint64_t a, uint64_t b) { return cdiv(a, b) * b; }

struct DBuf {
  void* p = nullptr;
  size_t cap = 0;
  bool ensure(size_t bytes) {
    if (p && bytes <= cap) return true;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    if (cudaMalloc(&p, bytes ? bytes : 16) != cudaSuccess) return false;
    cap = bytes ? bytes : 16;
    return true;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
  template <class T>
  T* as() const { return static_cast<T*>(p); }
};

// ============================================================== transports

enum Phase { kDot = 0, kLift = 1, kOt = 2, kMsb = 3, kOr = 4, kPhases = 5 };

struct Msg {
  int peer;      // party index 0..2
  void* buf;     // device memory
  size_t bytes;  // bytes on the wire
};

struct Transport {
  virtual ~Transport() = default;
  // One protocol step: all sends and receives, ordered on stream st.
  virtual std::string exchange(int self, const std::vector<Msg>& sends, const std::vector<Msg>& recvs,
                               cudaStream_t st) = 0;
};

struct NcclTransport : Transport {
  ncclComm_t comm = nullptr;
  ~NcclTransport() override {
    if (comm && nccl().ok) nccl().comm_destroy(comm);
  }
  std::string exchange(int, const std::vector<Msg>& sends, const std::vector<Msg>& recvs, cudaStream_t st) override {
    const NcclApi& n = nccl();
    ncclResult_t r = n.group_start();
    for (const Msg& m : sends)
      if (r == ncclSuccess && m.bytes) r = n.send(m.buf, m.bytes, ncclUint8, m.peer, comm, st);
    for (const Msg& m : recvs)
      if (r == ncclSuccess && m.bytes) r = n.recv(m.buf, m.bytes, ncclUint8, m.peer, comm, st);
    const ncclResult_t r2 = n.group_end();
    if (r != ncclSuccess) return std::string("nccl: ") + n.error_string(r);
    if (r2 != ncclSuccess) return std::string("nccl: ") + n.error_string(r2);
    return "";
  }
};

}  // namespace

// ---- in-process mailbox (three parties in one process, one host thread each)
struct irismpc_gpu_inproc {
  struct Item {
    void* buf;
    size_t bytes;
    cudaEvent_t ev;
  };
  std::mutex mu;
  std::condition_variable cv;
  std::deque<Item> q[3][3];  // [from][to]
};

namespace {

struct InProcTransport : Transport {
  irismpc_gpu_inproc* net = nullptr;
  std::string exchange(int self, const std::vector<Msg>& sends, const std::vector<Msg>& recvs,
                       cudaStream_t st) override {
    for (const Msg& m : sends) {
      irismpc_gpu_inproc::Item it{nullptr, m.bytes, nullptr};
      if (cudaMalloc(&it.buf, m.bytes ? m.bytes : 16) != cudaSuccess) return "inproc: oom";
      if (m.bytes) cudaMemcpyAsync(it.buf, m.buf, m.bytes, cudaMemcpyDeviceToDevice, st);
      cudaEventCreateWithFlags(&it.ev, cudaEventDisableTiming);
      cudaEventRecord(it.ev, st);
      std::lock_guard<std::mutex> g(net->mu);
      net->q[self][m.peer].push_back(it);
      net->cv.notify_all();
    }
    for (const Msg& m : recvs) {
      irismpc_gpu_inproc::Item it;
      {
        std::unique_lock<std::mutex> g(net->mu);
        auto& q = net->q[m.peer][self];
        if (!net->cv.wait_for(g, std::chrono::seconds(120), [&] { return !q.empty(); }))
          return "inproc: receive timed out";  // InProcNet::kTimeout
        it = q.front();
        q.pop_front();
      }
      if (it.bytes != m.bytes) return "inproc: bad payload size";
      cudaStreamWaitEvent(st, it.ev, 0);
      if (m.bytes) cudaMemcpyAsync(m.buf, it.buf, m.bytes, cudaMemcpyDeviceToDevice, st);
      cudaStreamSynchronize(st);
      cudaFree(it.buf);
      cudaEventDestroy(it.ev);
    }
    return "";
  }
};

// ============================================================== kernels

// 64-bit stream words [e, e + 8) of one seed, warp-cooperative like prf_window
// (the neighbour lane's block arrives by shuffle when e % 8 != 0).
__device__ __forceinline__ void prf_window64(const SeedKey& key, uint64_t e, bool next_contig, uint64_t out[8]) {
  uint32_t blk[16], nb[16];
  const uint64_t b = e / 8;
  chacha12_block(key, b, 0, blk);
  const int r = (int)(e % 8);
  if (r == 0) {
#pragma unroll
    for (int i = 0; i < 8; ++i) out[i] = chacha_word(blk, i);
    return;
  }
#pragma unroll
  for (int i = 0; i < 16; ++i) nb[i] = __shfl_down_sync(0xFFFFFFFFu, blk[i], 1);
  if (!next_contig) chacha12_block(key, b + 1, 0, nb);
  uint64_t w[16];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    w[i] = chacha_word(blk, i);
    w[8 + i] = chacha_word(nb, i);
  }
  switch (r) {  // warp-uniform: one static selection
#define SEL(R)                                   \
  case R:                                        \
    _Pragma("unroll") for (int i = 0; i < 8; ++i) out[i] = w[R + i]; \
    break;
    SEL(1) SEL(2) SEL(3) SEL(4) SEL(5) SEL(6)
    default:
#pragma unroll
      for (int i = 0; i < 8; ++i) out[i] = w[7 + i];
#undef SEL
  }
}

// reshare_pair<KH, KM> (engine.cpp:80-106, zero_ring<K> = low K bits of the
// u64 draws): own = z + F(seed_own) - F(seed_prev), hd at e = pos + i, ml at
// pos + n + i (KM > 0).  Writes the own components as u32 and the message in
// the reference's serialisation: n hd elements of HB bytes, then n ml elements
// of MB bytes.  Thread -> 8 lanes (warp-contiguous windows).
template <int HB, int MB>
__global__ void k_pty_reshare(const void* __restrict__ zh, const void* __restrict__ zm, uint64_t n, SeedKey own,
                              SeedKey prev, uint64_t pos_own, uint64_t pos_prev, uint32_t* __restrict__ out_h,
                              uint32_t* __restrict__ out_m, uint8_t* __restrict__ msg) {
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t L8 = t * 8;
  const uint64_t ngrp = cdiv(n, 8);
  if ((t & ~31ull) >= ngrp) return;  // whole warp past the end
  const bool next_contig = (t & 31) != 31;  // lane 31's neighbour window lives in the next warp
#pragma unroll
  for (int f = 0; f < 2; ++f) {
    const int B = f == 0 ? HB : MB;
    if (B == 0) continue;
    const uint64_t off = f == 0 ? 0 : n;
    uint32_t fo[8], fp[8];
    prf_window<1>(own, pos_own + off + L8, next_contig, fo);
    prf_window<1>(prev, pos_prev + off + L8, next_contig, fp);
    if (t >= ngrp) continue;
    uint32_t* o = f == 0 ? out_h : out_m;
    uint8_t* mg = msg + (f == 0 ? 0 : n * HB);
    const uint32_t kmask = B == 4 ? 0xFFFFFFFFu : 0xFFFFu;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint64_t j = L8 + i;
      if (j >= n) break;
      const uint32_t z = B == 4 ? static_cast<const uint32_t*>(f == 0 ? zh : zm)[j]
                                : static_cast<const uint16_t*>(f == 0 ? zh : zm)[j];
      const uint32_t v = (z + fo[i] - fp[i]) & kmask;
      o[j] = v;
      if (B == 4)
        reinterpret_cast<uint32_t*>(mg)[j] = v;
      else
        reinterpret_cast<uint16_t*>(mg)[j] = (uint16_t)v;
    }
  }
}

// the previous party's message -> its own components as u32 (our prev components)
template <int HB, int MB>
__global__ void k_pty_unpack(const uint8_t* __restrict__ msg, uint64_t n, uint32_t* __restrict__ prev_h,
                             uint32_t* __restrict__ prev_m) {
  const uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (j >= n) return;
  prev_h[j] = HB == 4 ? reinterpret_cast<const uint32_t*>(msg)[j] : reinterpret_cast<const uint16_t*>(msg)[j];
  if (MB) {
    const uint8_t* m = msg + n * HB;
    prev_m[j] = MB == 4 ? reinterpret_cast<const uint32_t*>(m)[j] : reinterpret_cast<const uint16_t*>(m)[j];
  }
}

// comparison input for the variants without the MPC lift (engine.hpp:77-120), per component:
//   const-lift / no-lift : ml32 = ml, diff = a ml - b hd (mod 2^32; const_lift(hd16, b) = b hd)
//   plain-mask           : diff = public_minus(ceil((1 - 2r) public_ml), hd) mod 2^16, the
//                          constant entering component 1 (own at P1, prev at P2, rep3.hpp:59-71)
__global__ void k_pty_cmp(int plain, const uint32_t* __restrict__ hd, const uint32_t* __restrict__ ml,
                          const uint16_t* __restrict__ pub, uint64_t n, uint32_t a, uint32_t b, double coef,
                          int add_t, uint32_t* __restrict__ ml32, uint32_t* __restrict__ diff) {
  const uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (j >= n) return;
  if (plain) {
    const uint32_t t = add_t ? (uint32_t)(int64_t)ceil(__dmul_rn(coef, (double)pub[j])) : 0u;
    diff[j] = (t - hd[j]) & 0xFFFFu;
    ml32[j] = 0;
  } else {
    ml32[j] = ml[j];
    diff[j] = a * ml[j] - b * hd[j];
  }
}

// share_split: K-bit lane values (own, prev components) -> bit rows
// rows[c][j][w], lane i = bit i % 64 of word i / 64 (circuits.hpp:152-172).
// Thread -> 32 lanes of one component: 32x32 SWAR transpose, one u32 half-word per row.
template <typename T, int K>
__global__ void k_pty_split(const T* __restrict__ own, const T* __restrict__ prev, uint64_t n, uint64_t W,
                            uint64_t* __restrict__ rows, uint64_t half_words) {
  // half_words: 2 x the chunk's words; the ones past the last lane are written as zeros
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (t >= 2 * half_words) return;
  const int c = (int)(t / half_words);
  const uint64_t g = t % half_words;
  const T* src = (c == 0 ? own : prev) + 32 * g;
  uint32_t a[32];
  const uint64_t left = 32 * g < n ? n - 32 * g : 0;
#pragma unroll
  for (int i = 0; i < 32; ++i) a[i] = (uint64_t)i < left ? (uint32_t)src[i] : 0u;
  transpose32(a);
  uint32_t* r32 = reinterpret_cast<uint32_t*>(rows);
#pragma unroll
  for (int j = 0; j < K; ++j) r32[((uint64_t)(c * K + j) * W) * 2 + g] = a[j];
}

// One AND layer (and_layer, circuits.hpp:92-131) at one party: for gate g,
// x = xa ^ xb, y = ya ^ yb (own and prev components, null rows are zero),
// z_own = x_o y_o ^ x_p y_o ^ x_o y_p ^ F(seed_own, eo + w) ^ F(seed_prev, ep + w),
// dead lanes of the last word masked.  Thread -> 8 words of one gate.
struct GateDesc {
  const uint64_t* xo[2];
  const uint64_t* xp[2];
  const uint64_t* yo[2];
  const uint64_t* yp[2];
  uint64_t* zo;
  uint64_t eo, ep;   // stream elements of word 0 (own / prev seed)
  uint64_t words;    // words of this gate
  uint64_t lanes;    // live lanes
};
constexpr int kMaxGates = 64;
struct GateBatch {
  GateDesc g[kMaxGates];
  uint32_t ngates;
  uint64_t wblocks_per_gate;  // ceil(max words / 8)
};

__device__ __forceinline__ uint64_t ld2(const uint64_t* const a[2], uint64_t w) {
  return (a[0] ? a[0][w] : 0ull) ^ (a[1] ? a[1][w] : 0ull);
}

__global__ void k_pty_and(const __grid_constant__ GateBatch B, SeedKey own, SeedKey prev) {
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t total = (uint64_t)B.ngates * B.wblocks_per_gate;
  if ((t & ~31ull) >= total) return;
  const uint64_t tq = t < total ? t : total - 1;
  const uint32_t gi = (uint32_t)(tq / B.wblocks_per_gate);
  const uint64_t wb = tq % B.wblocks_per_gate;
  const GateDesc& G = B.g[gi];
  const bool next_contig = (t & 31) != 31 && wb + 1 < B.wblocks_per_gate && t + 1 < total;
  uint64_t fo[8], fp[8];
  prf_window64(own, G.eo + 8 * wb, next_contig, fo);
  prf_window64(prev, G.ep + 8 * wb, next_contig, fp);
  if (t >= total) return;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint64_t w = 8 * wb + i;
    if (w >= G.words) break;
    const uint64_t xo = ld2(G.xo, w), xp = ld2(G.xp, w), yo = ld2(G.yo, w), yp = ld2(G.yp, w);
    uint64_t z = (xo & yo) ^ (xp & yo) ^ (xo & yp) ^ fo[i] ^ fp[i];
    if (w == G.words - 1 && (G.lanes % 64)) z &= (1ull << (G.lanes % 64)) - 1;
    G.zo[w] = z;
  }
}

// dst = a ^ b over `words` (b may be null); a list of such ops
struct XorOp {
  uint64_t* dst;
  const uint64_t* a;
  const uint64_t* b;
};
constexpr int kMaxOps = 132;
struct XorBatch {
  XorOp op[kMaxOps];
  uint32_t nops;
  uint64_t words;
};
__global__ void k_pty_xor(const __grid_constant__ XorBatch X) {
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (t >= (uint64_t)X.nops * X.words) return;
  const XorOp& o = X.op[t / X.words];
  const uint64_t w = t % X.words;
  o.dst[w] = o.a[w] ^ (o.b ? o.b[w] : 0ull);
}

// bit_inject<W> (convert.hpp:84-155), per role; thread -> 8 lanes with
// warp-cooperative stream windows (seed_1: 8 elements at e1 + L8, seed_3: 24
// elements (c3, w0, w1 per lane) at e3 + 3 L8).  bits: own/prev bit rows.
// role 0 (P1): out (c1, c3), msg[2i], msg[2i+1] = w0 ^ m0, w1 ^ m1 -> P2
// role 2 (P3): out own = c3, msg[i] = x2 ? w1 : w0 -> P2
__global__ void k_pty_inject_send(int role, const uint64_t* __restrict__ bo, const uint64_t* __restrict__ bp,
                                  uint64_t n, uint32_t mask, SeedKey own, SeedKey prev, uint64_t e1, uint64_t e3,
                                  uint16_t* __restrict__ out_o, uint16_t* __restrict__ out_p,
                                  uint16_t* __restrict__ msg) {
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t ngrp = cdiv(n, 8);
  if ((t & ~31ull) >= ngrp) return;
  const uint64_t L8 = 8 * t;
  const bool next_contig = (t & 31) != 31;
  const uint64_t wv = t < ngrp ? (bo[L8 / 64] >> (L8 % 64)) : 0, pv = t < ngrp ? (bp[L8 / 64] >> (L8 % 64)) : 0;
  uint32_t w3[24];
  prf_window<3>(role == 0 ? prev : own, e3 + 3 * L8, next_contig, w3);
  if (role == 0) {
    uint32_t c1[8];
    prf_window<1>(own, e1 + L8, next_contig, c1);
    if (t >= ngrp) return;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (L8 + i >= n) break;
      const uint32_t x1 = (uint32_t)(wv >> i) & 1u, x3 = (uint32_t)(pv >> i) & 1u;
      const uint32_t a1 = c1[i] & mask, c3 = w3[3 * i] & mask;
      const uint32_t m0 = ((0u ^ x1 ^ x3) - a1 - c3) & mask, m1 = ((1u ^ x1 ^ x3) - a1 - c3) & mask;
      msg[2 * (L8 + i)] = (uint16_t)((w3[3 * i + 1] ^ m0) & mask);
      msg[2 * (L8 + i) + 1] = (uint16_t)((w3[3 * i + 2] ^ m1) & mask);
      out_o[L8 + i] = (uint16_t)a1;
      out_p[L8 + i] = (uint16_t)c3;
    }
  } else {
    if (t >= ngrp) return;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (L8 + i >= n) break;
      const uint32_t x2 = (uint32_t)(pv >> i) & 1u;
      msg[L8 + i] = (uint16_t)((x2 ? w3[3 * i + 2] : w3[3 * i + 1]) & mask);
      out_o[L8 + i] = (uint16_t)(w3[3 * i] & mask);
    }
  }
}
// role 1 (P2): c1 from its prev stream, c2 = k_{x2} ^ w_{x2}; out (c2, c1); msg[i] = c2 -> P3
__global__ void k_pty_inject_p2(const uint64_t* __restrict__ bo, uint64_t n, uint32_t mask, SeedKey prev,
                                uint64_t e1, const uint16_t* __restrict__ ks, const uint16_t* __restrict__ ws,
                                uint16_t* __restrict__ out_o, uint16_t* __restrict__ out_p,
                                uint16_t* __restrict__ msg) {
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t ngrp = cdiv(n, 8);
  if ((t & ~31ull) >= ngrp) return;
  const uint64_t L8 = 8 * t;
  uint32_t c1[8];
  prf_window<1>(prev, e1 + L8, (t & 31) != 31, c1);
  if (t >= ngrp) return;
  const uint64_t wv = bo[L8 / 64] >> (L8 % 64);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    if (L8 + i >= n) break;
    const uint64_t j = L8 + i;
    const uint32_t x2 = (uint32_t)(wv >> i) & 1u;
    const uint32_t c2 = ((uint32_t)ks[2 * j + x2] ^ (uint32_t)ws[j]) & mask;
    msg[j] = (uint16_t)c2;
    out_o[j] = (uint16_t)c2;
    out_p[j] = (uint16_t)(c1[i] & mask);
  }
}

// lift output and comparison input per component (convert.hpp:169-192,
// engine.hpp:94-120): ml32 = ml - (inj17 << 17) - (inj16 << 16), diff = a ml32 - b hd
__global__ void k_pty_diff(const uint32_t* __restrict__ ml, const uint32_t* __restrict__ hd,
                           const uint16_t* __restrict__ i17, const uint16_t* __restrict__ i16, uint64_t n2,
                           uint32_t a, uint32_t b, uint32_t* __restrict__ ml32, uint32_t* __restrict__ diff) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;  // [comp][lane]
  if (i >= n2) return;
  const uint32_t m = (uint32_t)ml[i] - ((uint32_t)i17[i] << 17) - ((uint32_t)i16[i] << 16);
  ml32[i] = m;
  diff[i] = a * m - b * (uint32_t)hd[i];
}

// OR tree: gather each group's lanes of the MSB bit rows into its row
struct OrGroup {
  uint64_t len;        // lanes of the group
  uint64_t db_lane0;   // first DB lane (contiguous DB part)
  uint64_t db_len;     // DB lanes
  uint64_t pair_off;   // offset of its pair-lane list in `pairs`
  uint64_t row_off;    // word offset of its row in the pool
};
__global__ void k_pty_or_gather(const OrGroup* __restrict__ G, uint32_t ngroups, const uint64_t* __restrict__ pairs,
                                const uint64_t* __restrict__ mo, const uint64_t* __restrict__ mp,
                                uint64_t* __restrict__ pool_o, uint64_t* __restrict__ pool_p, uint64_t max_words) {
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (t >= (uint64_t)ngroups * max_words) return;
  const OrGroup g = G[t / max_words];
  const uint64_t w = t % max_words;
  if (w * 64 >= g.len) return;
  uint64_t o = 0, p = 0;
  for (int b = 0; b < 64; ++b) {
    const uint64_t i = w * 64 + b;
    if (i >= g.len) break;
    const uint64_t ln = i < g.db_len ? g.db_lane0 + i : pairs[g.pair_off + (i - g.db_len)];
    o |= ((mo[ln / 64] >> (ln % 64)) & 1ull) << b;
    p |= ((mp[ln / 64] >> (ln % 64)) & 1ull) << b;
  }
  pool_o[g.row_off + w] = o;
  pool_p[g.row_off + w] = p;
}

// one or_tree_batch level: lo = lanes [0, na), hi = lanes [na, len)
struct OrLevel {
  uint64_t src_off, dst_off, na, nb, wa, wb;
  uint64_t t_off;   // word offset into the AND output (concatenated over groups)
  uint64_t eo, ep;  // stream elements (own / prev seed) of its first AND word
};
__device__ __forceinline__ uint64_t hi_word(const uint64_t* row, uint64_t na, uint64_t nb, uint64_t w) {
  const uint64_t bit = na + 64 * w;
  if (64 * w >= nb) return 0;
  const uint64_t q = bit / 64, r = bit % 64;
  uint64_t v = row[q] >> r;
  if (r && 64 * w + (64 - r) < nb) v |= row[q + 1] << (64 - r);
  const uint64_t left = nb - 64 * w;
  if (left < 64) v &= (1ull << left) - 1;
  return v;
}
__global__ void k_pty_or_and(const OrLevel* __restrict__ L, uint32_t nl, uint64_t max_wb, const uint64_t* __restrict__ po,
                             const uint64_t* __restrict__ pp, SeedKey own, SeedKey prev, uint64_t* __restrict__ tz) {
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (t >= (uint64_t)nl * max_wb) return;
  const OrLevel l = L[t / max_wb];
  const uint64_t w = t % max_wb;
  if (w >= l.wb) return;
  const uint64_t lo_o = po[l.src_off + w], lo_p = pp[l.src_off + w];
  const uint64_t hi_o = hi_word(po + l.src_off, l.na, l.nb, w), hi_p = hi_word(pp + l.src_off, l.na, l.nb, w);
  uint32_t blk[16];
  chacha12_block(own, (l.eo + w) / 8, 0, blk);
  const uint64_t fo = chacha_word(blk, (int)((l.eo + w) % 8));
  chacha12_block(prev, (l.ep + w) / 8, 0, blk);
  const uint64_t fp = chacha_word(blk, (int)((l.ep + w) % 8));
  uint64_t z = (lo_o & hi_o) ^ (lo_p & hi_o) ^ (lo_o & hi_p) ^ fo ^ fp;
  if (w == l.wb - 1 && (l.nb % 64)) z &= (1ull << (l.nb % 64)) - 1;
  tz[l.t_off + w] = z;
}
// fold: new = lo ^ hi ^ t over wa words, both components
__global__ void k_pty_or_fold(const OrLevel* __restrict__ L, uint32_t nl, uint64_t max_wa, uint64_t* __restrict__ po,
                              uint64_t* __restrict__ pp, const uint64_t* __restrict__ to,
                              const uint64_t* __restrict__ tp, uint64_t* __restrict__ qo, uint64_t* __restrict__ qp) {
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (t >= (uint64_t)nl * max_wa) return;
  const OrLevel l = L[t / max_wa];
  const uint64_t w = t % max_wa;
  if (w >= l.wa) return;
  uint64_t lo_o = po[l.src_off + w], lo_p = pp[l.src_off + w];
  const uint64_t rem = l.na - 64 * w;  // lo has na lanes
  if (rem < 64) {
    lo_o &= (1ull << rem) - 1;
    lo_p &= (1ull << rem) - 1;
  }
  const uint64_t ho = hi_word(po + l.src_off, l.na, l.nb, w), hp = hi_word(pp + l.src_off, l.na, l.nb, w);
  const uint64_t tzo = w < l.wb ? to[l.t_off + w] : 0, tzp = w < l.wb ? tp[l.t_off + w] : 0;
  qo[l.dst_off + w] = lo_o ^ ho ^ tzo;
  qp[l.dst_off + w] = lo_p ^ hp ^ tzp;
}

// pack bit 0 of group rows (or any word rows) into bytes for open_bits_to
__global__ void k_pty_pack_groups(const uint64_t* __restrict__ pool, const uint64_t* __restrict__ row_off,
                                  uint32_t ngroups, uint8_t* __restrict__ out) {
  const uint32_t byte = blockIdx.x * blockDim.x + threadIdx.x;
  if (byte >= (ngroups + 7) / 8) return;
  uint32_t v = 0;
  for (int b = 0; b < 8; ++b) {
    const uint32_t g = byte * 8 + b;
    if (g < ngroups && row_off[g] != ~0ull) v |= (uint32_t)(pool[row_off[g]] & 1ull) << b;
  }
  out[byte] = (uint8_t)v;
}

}  // namespace

// ============================================================== context

struct PartyField {
  FieldFmt fmt{};
  uint32_t slots = 1;  // DB planes: own (+ prev for replicated)
  uint32_t nseg = 1;
  DBuf db, q, qa, pc;
  CUtensorMap tA, tB, tQA;
  uint32_t ncols_pad_cur = 0;
  uint64_t qa_spad = 0;
};

struct irismpc_gpu_party {
  irismpc_gpu_config cfg{};
  int p = 0;  // 0..2
  int shamir = 0;
  int variant = kMpcLift;
  VariantWidths vw{16, 16, 32};
  uint32_t l = 0, l_pad = 0;
  uint64_t rec = 0;
  SeedKey own{}, prev{};
  uint64_t pos[2] = {0, 0};  // stream positions of seed_own, seed_prev
  Transport* net = nullptr;
  cudaStream_t st = nullptr;
  cudaEvent_t ev[2];
  cudaEvent_t pev[6];  // phase boundaries
  // comparison-phase pipeline: lane chunks compute on cs[k] while the comm
  // stream carries the other chunk's messages (same order at every party)
  cudaStream_t cst = nullptr, cs[2] = {nullptr, nullptr};
  cudaEvent_t ea[2], eb[2], ej[3];
  PartyField fld[2];
  uint64_t s = 0, s_pad = 0;
  bool db_loaded = false;
  std::string err;
  uint64_t led_bytes[kPhases] = {0, 0, 0, 0, 0}, led_rounds[kPhases] = {0, 0, 0, 0, 0}, wire = 0;
  std::vector<cudaEvent_t> xev;  // exchange start/stop pairs of the current query (profiling)
  size_t nxev = 0;
  // work buffers
  DBuf qpay, dots, rs, rows, carry, chain, zbuf, zrecv, inj, msg, msg2, ml32, diff, bits, pairs, groups, levels,
      pool[2], tz[2], rowoff, open_buf[3], xsend, xrecv, c2buf;
  uint64_t tap_n = 0;
};

namespace {

int pfail(irismpc_gpu_party* c, int code, const std::string& m) {
  if (c) c->err = m;
  return code;
}
#define PCK(c, x)                                                                                        \
  do {                                                                                                   \
    cudaError_t e_ = (x);                                                                                \
    if (e_ != cudaSuccess) return pfail(c, IRISMPC_GPU_ERR_DEVICE, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

int next_of(int p) { return (p + 1) % 3; }
int prev_of(int p) { return (p + 2) % 3; }

// one lane chunk of the pipelined comparison phase
struct Chunk {
  int idx;             // 0 counts the protocol rounds
  uint64_t w0, words;  // 64-lane words [w0, w0 + words)
  uint64_t lane0, lanes;
  cudaStream_t st;     // compute stream
};

// one protocol step through the transport + the ledger (counted bytes per the
// reference's serialisation; rounds per ctx.comm.round call of that phase).
// On a chunk stream the message hops to the comm stream and back, so this
// chunk's transfer overlaps the other chunk's kernels.
int step_on(irismpc_gpu_party* c, cudaStream_t cs, bool count_rounds, Phase ph, const std::vector<Msg>& sends,
            const std::vector<Msg>& recvs, const std::vector<uint64_t>& counted, uint32_t rounds) {
  for (size_t i = 0; i < sends.size(); ++i) {
    c->led_bytes[ph] += i < counted.size() ? counted[i] : sends[i].bytes;
    c->wire += sends[i].bytes;
  }
  if (count_rounds) c->led_rounds[ph] += rounds;
  while (c->xev.size() < c->nxev + 2) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    c->xev.push_back(e);
  }
  cudaStream_t xs = cs;
  int k = -1;
  if (cs != c->st) {
    k = cs == c->cs[0] ? 0 : 1;
    cudaEventRecord(c->ea[k], cs);
    cudaStreamWaitEvent(c->cst, c->ea[k], 0);
    xs = c->cst;
  }
  cudaEventRecord(c->xev[c->nxev], xs);
  const std::string e = c->net->exchange(c->p, sends, recvs, xs);
  cudaEventRecord(c->xev[c->nxev + 1], xs);
  c->nxev += 2;
  if (k >= 0) {
    cudaEventRecord(c->eb[k], c->cst);
    cudaStreamWaitEvent(cs, c->eb[k], 0);
  }
  if (!e.empty()) return pfail(c, IRISMPC_GPU_ERR_DEVICE, e);
  return 0;
}

int step(irismpc_gpu_party* c, Phase ph, const std::vector<Msg>& sends, const std::vector<Msg>& recvs,
         const std::vector<uint64_t>& counted, uint32_t rounds) {
  return step_on(c, c->st, true, ph, sends, recvs, counted, rounds);
}

int party_init(const irismpc_gpu_config* cfg, uint32_t party, irismpc_gpu_party** out, std::string* why) {
  if (!cfg || !out || party < 1 || party > 3) return IRISMPC_GPU_ERR_CONFIG;
  if (cfg->variant > IRISMPC_GPU_VARIANT_NO_LIFT) {
    *why = "unknown variant";
    return IRISMPC_GPU_ERR_CONFIG;
  }
  // EngineConfig::validate (engine.cpp:21-34)
  if (cfg->backend > 1) return IRISMPC_GPU_ERR_CONFIG;
  if (cfg->l == 0 || cfg->l % 8 != 0 || cfg->a > cfg->b || cfg->rotations % 2 == 0) return IRISMPC_GPU_ERR_BOUNDS;
  if (cfg->variant == IRISMPC_GPU_VARIANT_PLAIN_MASK) {
    const uint64_t t = 1ull << 16;
    if (!(cfg->l < t / 4 && cfg->l < t - (t >> 1))) return IRISMPC_GPU_ERR_BOUNDS;
  } else {
    if (cfg->m != 16 || cfg->b != (1u << 16)) return IRISMPC_GPU_ERR_BOUNDS;
    const uint64_t t = 1ull << 32, bl = (uint64_t)cfg->b * cfg->l;
    if (!(bl < t / 4 && bl < t - (t >> 1))) return IRISMPC_GPU_ERR_BOUNDS;
  }
  if (cfg->rotations > 31) return IRISMPC_GPU_ERR_CONFIG;
  if (cfg->backend == IRISMPC_GPU_BACKEND_SHAMIR && cfg->rotations > 1 && (cfg->l / 64) % 2 != 0)
    return IRISMPC_GPU_ERR_BOUNDS;
  if (cudaSetDevice(cfg->device) != cudaSuccess) return IRISMPC_GPU_ERR_DEVICE;
  auto* c = new irismpc_gpu_party;
  c->cfg = *cfg;
  c->p = (int)party - 1;
  c->shamir = cfg->backend == IRISMPC_GPU_BACKEND_SHAMIR;
  c->l = cfg->l;
  c->l_pad = (uint32_t)rup(cfg->l, kGemmBK);
  c->rec = irismpc_gpu_record_bytes(cfg->backend, cfg->variant, cfg->l);
  std::memcpy(c->own.k, cfg->seeds, 16);
  std::memcpy(c->prev.k, cfg->seeds + 16, 16);
  c->variant = (int)cfg->variant;
  c->vw = variant_widths(c->variant);
  const int widths[2] = {c->vw.kh / 8, c->vw.km / 8};  // 0: public mask bits
  const uint64_t code_b = (uint64_t)(c->shamir ? cfg->l : 2 * cfg->l) * widths[0];
  for (int fi = 0; fi < 2; ++fi) {
    PartyField& f = c->fld[fi];
    f.fmt.rec_bytes = c->rec;
    f.fmt.off = fi == 0 ? 0 : code_b;
    f.fmt.width = widths[fi];
    f.fmt.limbs = widths[fi] ? widths[fi] : 1;
    f.slots = (widths[fi] && !c->shamir) ? 2 : 1;
    f.nseg = (widths[fi] && !c->shamir) ? 2 : 1;
  }
  if (cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking) != cudaSuccess) {
    delete c;
    return IRISMPC_GPU_ERR_DEVICE;
  }
  cudaEventCreate(&c->ev[0]);
  cudaEventCreate(&c->ev[1]);
  for (auto& e : c->pev) cudaEventCreate(&e);
  cudaStreamCreateWithFlags(&c->cst, cudaStreamNonBlocking);
  for (auto& x : c->cs) cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking);
  for (auto& e : c->ea) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  for (auto& e : c->eb) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  for (auto& e : c->ej) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  // lambda_p for the Shamir parse (the same constants as the 3-party context)
  uint32_t lam[6] = {1, 2, 0xFFFFFFFFu, 0xFFFFFFFEu, 1, 0};  // 1+2X, -(1+2X), 1 (galois.hpp:124-128)
  set_lambda(lam);
  *out = c;
  return 0;
}

// parse one payload (rows of this party's records) into a field's planes
void parse_party_rows(irismpc_gpu_party* c, PartyField& f, const uint8_t* pay, uint64_t rows, uint64_t s_pad,
                      uint8_t* planes) {
  FieldFmt fo = f.fmt;
  fo.slot = 0;
  launch_parse_field(pay, rows, 0, c->l, c->l_pad, s_pad, c->p, c->shamir, fo, planes, c->st);
  if (!c->shamir && f.fmt.width) {
    FieldFmt fp = f.fmt;
    fp.slot = 1;
    fp.take_prev = 1;
    launch_parse_field(pay, rows, 0, c->l, c->l_pad, s_pad, c->p, c->shamir, fp, planes, c->st);
  }
}

// bit_extract_sum over summand rows X (own/prev components of summand p and
// p-1 only, share_split) for instances `idx`, rows j >= K zero.  Gate g of the
// call uses stream elements base[own|prev] + g W + w (w global).  Results ->
// res_o/res_p rows [inst][W].  Rows are full width; every round runs once per
// lane chunk (on the chunk's stream), so the chunks' transfers and kernels overlap.
int bit_extract(irismpc_gpu_party* c, Phase ph, const uint64_t* Xo, const uint64_t* Xp, int K,
                const std::vector<int>& idx, const std::vector<Chunk>& chunks, uint64_t /*n: lanes, the chunks carry them*/,
                uint64_t W, uint64_t base_o, uint64_t base_p, uint64_t* res_o, uint64_t* res_p) {
  const int p = c->p;
  const int ninst = (int)idx.size();
  int maxm = 0;
  for (int m : idx) maxm = std::max(maxm, m);
  auto XR = [&](int comp, int j) -> const uint64_t* {  // own / prev component of summand row j
    if (j >= K) return nullptr;
    return (comp == 0 ? Xo : Xp) + (uint64_t)j * W;
  };
  // component views of a_k_j: own comp nonzero iff k == p, prev iff k == p - 1
  auto A = [&](int k, int comp, int j) -> const uint64_t* {
    if (comp == 0) return k == p ? XR(0, j) : nullptr;
    return k == prev_of(p) ? XR(1, j) : nullptr;
  };
  auto off = [](const uint64_t* r, uint64_t w0) -> const uint64_t* { return r ? r + w0 : nullptr; };
  int total_fa = 0;
  for (int m : idx) total_fa += m;
  const int maxg = std::max(total_fa, ninst);
  if (!c->carry.ensure(2ull * total_fa * W * 8 + 16) || !c->chain.ensure(2ull * ninst * W * 8 + 16) ||
      !c->zbuf.ensure((uint64_t)maxg * W * 8 + 16) || !c->zrecv.ensure((uint64_t)maxg * W * 8 + 16))
    return pfail(c, IRISMPC_GPU_ERR_DEVICE, "oom (bit extract)");
  uint64_t* carry = c->carry.as<uint64_t>();  // [comp][fa gate][W]
  uint64_t* chain = c->chain.as<uint64_t>();  // [comp][inst][W]
  auto carry_row = [&](int comp, int g) { return carry + ((uint64_t)comp * total_fa + g) * W; };
  auto chain_row = [&](int comp, int k) { return chain + ((uint64_t)comp * ninst + k) * W; };
  std::vector<int> fa0(ninst);
  {
    int gi = 0;
    for (int k = 0; k < ninst; ++k) {
      fa0[k] = gi;
      gi += idx[k];
    }
  }
  // per chunk: a contiguous z area [gates][words] at maxg * w0
  auto zarea = [&](uint64_t* z, const Chunk& ch) { return z + (uint64_t)maxg * ch.w0; };
  uint64_t g = 0;
  // ---- FA layer: one round, gates in instance order then j
  for (const Chunk& ch : chunks) {
    GateBatch B{};
    uint64_t* zo = zarea(c->zbuf.as<uint64_t>(), ch);
    uint64_t* zp = zarea(c->zrecv.as<uint64_t>(), ch);
    int gi = 0;
    for (int k = 0; k < ninst; ++k)
      for (int j = 0; j < idx[k]; ++j, ++gi) {
        GateDesc& d = B.g[gi];
        // t1 = a0 ^ a2, t2 = a1 ^ a2
        d.xo[0] = off(A(0, 0, j), ch.w0); d.xo[1] = off(A(2, 0, j), ch.w0);
        d.xp[0] = off(A(0, 1, j), ch.w0); d.xp[1] = off(A(2, 1, j), ch.w0);
        d.yo[0] = off(A(1, 0, j), ch.w0); d.yo[1] = off(A(2, 0, j), ch.w0);
        d.yp[0] = off(A(1, 1, j), ch.w0); d.yp[1] = off(A(2, 1, j), ch.w0);
        d.zo = zo + (uint64_t)gi * ch.words;
        d.eo = base_o + (g + gi) * W + ch.w0;
        d.ep = base_p + (g + gi) * W + ch.w0;
        d.words = ch.words;
        d.lanes = ch.lanes;
      }
    B.ngates = (uint32_t)gi;
    B.wblocks_per_gate = cdiv(ch.words, 8);
    k_pty_and<<<nblk(rup((uint64_t)gi * B.wblocks_per_gate, 32)), kThreads, 0, ch.st>>>(B, c->own, c->prev);
    PCK(c, cudaGetLastError());
    int rc = step_on(c, ch.st, ch.idx == 0, ph, {{next_of(p), zo, (size_t)gi * ch.words * 8}},
                     {{prev_of(p), zp, (size_t)gi * ch.words * 8}}, {(uint64_t)gi * cdiv(ch.lanes, 8)}, 1);
    if (rc) return rc;
    // carry = z ^ a2
    XorBatch ops{};
    ops.words = ch.words;
    for (int q = 0; q < gi; ++q) {
      int k = 0;
      while (k + 1 < ninst && fa0[k + 1] <= q) ++k;
      const int j = q - fa0[k];
      ops.op[ops.nops++] = {carry_row(0, q) + ch.w0, zo + (uint64_t)q * ch.words, off(A(2, 0, j), ch.w0)};
      ops.op[ops.nops++] = {carry_row(1, q) + ch.w0, zp + (uint64_t)q * ch.words, off(A(2, 1, j), ch.w0)};
    }
    k_pty_xor<<<nblk((uint64_t)ops.nops * ch.words), kThreads, 0, ch.st>>>(ops);
  }
  g += total_fa;
  // ---- ripple chain: round t, gates in instance order (circuits.hpp:263-288)
  for (int t = 1; t + 1 <= maxm; ++t) {
    std::vector<int> which;
    for (int k = 0; k < ninst; ++k)
      if (t + 1 <= idx[k]) which.push_back(k);
    const int gn = (int)which.size();
    for (const Chunk& ch : chunks) {
      GateBatch B{};
      uint64_t* zo = zarea(c->zbuf.as<uint64_t>(), ch);
      uint64_t* zp = zarea(c->zrecv.as<uint64_t>(), ch);
      for (int gi = 0; gi < gn; ++gi) {
        const int k = which[gi];
        GateDesc& d = B.g[gi];
        const int cg = fa0[k] + (t - 1);  // carry_{t-1}
        if (t == 1) {
          d.xo[0] = off(XR(0, t), ch.w0); d.xp[0] = off(XR(1, t), ch.w0);  // s_1 (own comp = X row)
          d.yo[0] = carry_row(0, cg) + ch.w0; d.yp[0] = carry_row(1, cg) + ch.w0;
        } else {
          d.xo[0] = off(XR(0, t), ch.w0); d.xo[1] = chain_row(0, k) + ch.w0;
          d.xp[0] = off(XR(1, t), ch.w0); d.xp[1] = chain_row(1, k) + ch.w0;
          d.yo[0] = carry_row(0, cg) + ch.w0; d.yo[1] = chain_row(0, k) + ch.w0;
          d.yp[0] = carry_row(1, cg) + ch.w0; d.yp[1] = chain_row(1, k) + ch.w0;
        }
        d.zo = zo + (uint64_t)gi * ch.words;
        d.eo = base_o + (g + gi) * W + ch.w0;
        d.ep = base_p + (g + gi) * W + ch.w0;
        d.words = ch.words;
        d.lanes = ch.lanes;
      }
      B.ngates = (uint32_t)gn;
      B.wblocks_per_gate = cdiv(ch.words, 8);
      k_pty_and<<<nblk(rup((uint64_t)gn * B.wblocks_per_gate, 32)), kThreads, 0, ch.st>>>(B, c->own, c->prev);
      PCK(c, cudaGetLastError());
      int rc = step_on(c, ch.st, ch.idx == 0, ph, {{next_of(p), zo, (size_t)gn * ch.words * 8}},
                       {{prev_of(p), zp, (size_t)gn * ch.words * 8}}, {(uint64_t)gn * cdiv(ch.lanes, 8)}, 1);
      if (rc) return rc;
      XorBatch ops{};
      ops.words = ch.words;
      for (int q = 0; q < gn; ++q) {
        const int k = which[q];
        ops.op[ops.nops++] = {chain_row(0, k) + ch.w0, zo + (uint64_t)q * ch.words,
                              t == 1 ? nullptr : chain_row(0, k) + ch.w0};
        ops.op[ops.nops++] = {chain_row(1, k) + ch.w0, zp + (uint64_t)q * ch.words,
                              t == 1 ? nullptr : chain_row(1, k) + ch.w0};
      }
      k_pty_xor<<<nblk((uint64_t)ops.nops * ch.words), kThreads, 0, ch.st>>>(ops);
    }
    g += gn;
  }
  // ---- result_k = s_m ^ carry_{m-1} ^ chain (m >= 2): two passes (the second XORs in place)
  for (const Chunk& ch : chunks) {
    XorBatch first{}, second{};
    first.words = second.words = ch.words;
    for (int k = 0; k < ninst; ++k) {
      const int m = idx[k];
      for (int comp = 0; comp < 2; ++comp) {
        uint64_t* dst = (comp == 0 ? res_o : res_p) + (uint64_t)k * W + ch.w0;
        first.op[first.nops++] = {dst, carry_row(comp, fa0[k] + m - 1) + ch.w0,
                                  m >= 2 ? chain_row(comp, k) + ch.w0 : nullptr};
        if (const uint64_t* sm = XR(comp, m)) second.op[second.nops++] = {dst, dst, sm + ch.w0};
      }
    }
    k_pty_xor<<<nblk((uint64_t)first.nops * ch.words), kThreads, 0, ch.st>>>(first);
    if (second.nops) k_pty_xor<<<nblk((uint64_t)second.nops * ch.words), kThreads, 0, ch.st>>>(second);
  }
  PCK(c, cudaGetLastError());
  return 0;
}

// bit_inject<Wd> of bit rows (bo, bp) -> out own/prev u16 components; per
// lane chunk, the 3-OT's two rounds (P1 -> P2 and P3 -> P2, then P2 -> P3)
int bit_inject(irismpc_gpu_party* c, const uint64_t* bo, const uint64_t* bp, const std::vector<Chunk>& chunks,
               uint64_t n, int Wd, uint64_t e1, uint64_t e3, uint16_t* out_o, uint16_t* out_p) {
  const int p = c->p;
  const uint32_t mask = (1u << Wd) - 1;
  const size_t eb = 2;  // Ring<15>, Ring<16>: 2-byte elements
  if (!c->msg.ensure(2 * n * eb + 16) || !c->msg2.ensure(2 * n * eb + 16) || !c->c2buf.ensure(n * eb + 16))
    return pfail(c, IRISMPC_GPU_ERR_DEVICE, "oom (inject)");
  int rc = 0;
  for (const Chunk& ch : chunks) {
    const uint64_t L = ch.lane0, m = ch.lanes;
    const bool first = ch.idx == 0;
    const uint64_t* cbo = bo + ch.w0;
    const uint64_t* cbp = bp + ch.w0;
    uint16_t* m1 = c->msg.as<uint16_t>() + 2 * L;
    uint16_t* m2 = c->msg2.as<uint16_t>() + L;
    const unsigned gr = nblk(rup(cdiv(m, 8), 32));
    if (p == 0) {  // P1: sender
      k_pty_inject_send<<<gr, kThreads, 0, ch.st>>>(0, cbo, cbp, m, mask, c->own, c->prev, e1 + L, e3 + 3 * L,
                                                     out_o + L, out_p + L, m1);
      rc = step_on(c, ch.st, first, kOt, {{1, m1, 2 * m * eb}}, {}, {}, 1);
      if (!rc) rc = step_on(c, ch.st, first, kOt, {}, {}, {}, 1);  // c_2 forwarding stage, party 1 idle
    } else if (p == 2) {  // P3: helper
      k_pty_inject_send<<<gr, kThreads, 0, ch.st>>>(2, cbo, cbp, m, mask, c->own, c->prev, e1 + L, e3 + 3 * L,
                                                     out_o + L, out_p + L, m1);
      rc = step_on(c, ch.st, first, kOt, {{1, m1, m * eb}}, {}, {}, 1);
      if (!rc) rc = step_on(c, ch.st, first, kOt, {}, {{1, out_p + L, m * eb}}, {}, 1);  // c_2 -> prev component
    } else {  // P2: receiver
      rc = step_on(c, ch.st, first, kOt, {}, {{0, m1, 2 * m * eb}, {2, m2, m * eb}}, {}, 1);
      if (rc) return rc;
      uint16_t* c2 = c->c2buf.as<uint16_t>() + L;
      k_pty_inject_p2<<<gr, kThreads, 0, ch.st>>>(cbo, m, mask, c->prev, e1 + L, m1, m2, out_o + L, out_p + L, c2);
      rc = step_on(c, ch.st, first, kOt, {{2, c2, m * eb}}, {}, {}, 1);
    }
    if (rc) return rc;
  }
  PCK(c, cudaGetLastError());
  return 0;
}

// open packed bits to P1 (open_bits_to, circuits.hpp:449-486); P1 gets `out`
int open_to_p1(irismpc_gpu_party* c, const uint8_t* own_bytes, const uint8_t* prev_bytes, uint64_t lanes,
               uint8_t* out_host) {
  const uint64_t bytes = cdiv(lanes, 8);
  const int p = c->p;
  if (p == 0) {
    if (!c->open_buf[0].ensure(bytes + 16) || !c->open_buf[1].ensure(bytes + 16))
      return pfail(c, IRISMPC_GPU_ERR_DEVICE, "oom (open)");
    int rc = step(c, kOr, {}, {{1, c->open_buf[0].p, bytes}, {2, c->open_buf[1].p, bytes}}, {}, 1);
    if (rc) return rc;
    std::vector<uint8_t> a(bytes), b(bytes), mo(bytes), mp(bytes);
    PCK(c, cudaMemcpyAsync(a.data(), c->open_buf[0].p, bytes, cudaMemcpyDeviceToHost, c->st));
    PCK(c, cudaMemcpyAsync(b.data(), c->open_buf[1].p, bytes, cudaMemcpyDeviceToHost, c->st));
    PCK(c, cudaMemcpyAsync(mo.data(), own_bytes, bytes, cudaMemcpyDeviceToHost, c->st));
    PCK(c, cudaMemcpyAsync(mp.data(), prev_bytes, bytes, cudaMemcpyDeviceToHost, c->st));
    PCK(c, cudaStreamSynchronize(c->st));
    if (a != b) return pfail(c, IRISMPC_GPU_ERR_INCONSISTENT, "open_bits_to: cross-check failed");
    for (uint64_t i = 0; i < lanes; ++i) out_host[i] = (uint8_t)(((mo[i / 8] ^ mp[i / 8] ^ a[i / 8]) >> (i % 8)) & 1);
    return 0;
  }
  // P2 (next of P1) sends its own component, P3 its prev
  const uint8_t* src = p == 1 ? own_bytes : prev_bytes;
  return step(c, kOr, {{0, const_cast<uint8_t*>(src), bytes}}, {}, {}, 1);
}

uint64_t ref_or_draws(uint64_t groups, uint64_t len, uint64_t* rounds) {
  uint64_t d = 0, r = 0;
  while (len > 1) {
    const uint64_t na = (len + 1) / 2, nb = len - na;
    d += groups * cdiv(nb, 64);
    len = na;
    ++r;
  }
  if (rounds) *rounds = r;
  return d;
}

int party_query(irismpc_gpu_party* c, const uint8_t* hq, size_t qlen, uint32_t persons, int membership,
                uint8_t* match_out, uint8_t* row_bits_out, irismpc_gpu_party_stats* stats) {
  if (!c->db_loaded) return pfail(c, IRISMPC_GPU_ERR_CONFIG, "no database loaded");
  const uint32_t ncodes = membership ? 1u : 2u * persons;
  if (qlen % c->rec != 0) return pfail(c, IRISMPC_GPU_ERR_CONFIG, "query payload size mismatch");
  if (qlen / c->rec != ncodes)
    return pfail(c, IRISMPC_GPU_ERR_CONFIG,
                 membership ? "membership expects exactly one query code" : "batch query expects 2 codes per person");
  for (auto& x : c->led_bytes) x = 0;
  for (auto& x : c->led_rounds) x = 0;
  c->wire = 0;
  c->nxev = 0;
  const int p = c->p;
  const uint32_t r = membership ? 1u : c->cfg.rotations;
  const uint64_t S = c->s, ncols = (uint64_t)ncodes * r;
  const uint32_t ncols_pad = (uint32_t)rup(ncols ? ncols : 1, kGemmBN);
  const uint64_t npairs = membership ? 0 : (uint64_t)persons * (persons ? persons - 1 : 0) / 2 * 4 * r;
  const uint64_t n = ncols * S + npairs;
  const uint64_t W = cdiv(n, 64);
  const uint32_t ngroups = membership ? 1u : persons;
  const int ko = p, kp = prev_of(p);  // seed indices of own / prev
  cudaStream_t st = c->st;
  PCK(c, cudaEventRecord(c->ev[0], st));
  // ---- payload + planes
  if (!c->qpay.ensure(qlen)) return pfail(c, IRISMPC_GPU_ERR_DEVICE, "oom (query)");
  PCK(c, cudaMemcpyAsync(c->qpay.p, hq, qlen, cudaMemcpyHostToDevice, st));
  const uint8_t* dq = c->qpay.as<uint8_t>();
  const VariantWidths vw = c->vw;
  const int V = c->variant;
  const int hb = c->fld[0].fmt.limbs == 4 ? 4 : 2, mb = c->fld[1].fmt.limbs == 4 ? 4 : 2;  // dot element bytes
  const uint64_t nml = vw.km ? n : 0;
  if (!c->dots.ensure((n + 8) * (hb + mb) + 64) || !c->rs.ensure(4 * (n + 8) * 4 + 64))
    return pfail(c, IRISMPC_GPU_ERR_DEVICE, "oom (dots)");
  uint8_t* dh = c->dots.as<uint8_t>();
  uint8_t* dm = dh + rup((n + 8) * hb, 16);
  for (int fi = 0; fi < 2; ++fi) {
    PartyField& f = c->fld[fi];
    const uint32_t L = (uint32_t)f.fmt.limbs, bn = gemm_bn(L);
    const int eb = L == 4 ? 4 : 2;
    const uint64_t rows = 3ull * f.nseg * L * ncols_pad;
    if (ncols_pad != f.ncols_pad_cur) {
      if (!f.q.ensure(rows * c->l_pad)) return pfail(c, IRISMPC_GPU_ERR_DEVICE, "oom (query planes)");
      PCK(c, cudaMemsetAsync(f.q.p, 0, rows * c->l_pad, st));
      if (make_plane_tmap(&f.tB, f.q.p, rows, c->l_pad, bn / 2))
        return pfail(c, IRISMPC_GPU_ERR_DEVICE, "tensor map (query)");
      f.ncols_pad_cur = ncols_pad;
    }
    // B planes of this party's payload (problem 0; the kernel also fills 1, 2 from the same bytes)
    launch_parse_query_field(dq, dq, dq, ncodes, c->l, c->l_pad, r, ncols_pad, c->shamir, f.fmt, f.q.as<uint8_t>(), st);
    uint8_t* out = fi == 0 ? dh : dm;
    if (S) {
      GemmArgs g{};
      g.s_pad = (uint32_t)c->s_pad;
      g.nb_rows = ncols_pad;
      g.nkb_seg = c->l_pad / kGemmBK;
      g.nseg = f.nseg;
      g.rep = f.nseg == 2;
      g.nprob = 1;
      g.limbs = L;
      g.s_valid = (uint32_t)S;
      g.ncols = (uint32_t)ncols;
      g.out = out;
      g.out_pstride = ncols * S;
      g.out_cstride = (uint32_t)S;
      launch_gemm(f.tA, f.tB, g, (uint32_t)(c->s_pad / kGemmBM), (uint32_t)cdiv(ncols, bn), st);
    }
    if (npairs) {
      const uint64_t spq = rup(ncodes, 2 * kGemmBM);
      const uint64_t arows = (uint64_t)f.slots * L * spq;
      if (spq != f.qa_spad) {
        if (!f.qa.ensure(arows * c->l_pad)) return pfail(c, IRISMPC_GPU_ERR_DEVICE, "oom (pair planes)");
        PCK(c, cudaMemsetAsync(f.qa.p, 0, arows * c->l_pad, st));
        if (make_plane_tmap(&f.tQA, f.qa.p, arows, c->l_pad, kGemmBM))
          return pfail(c, IRISMPC_GPU_ERR_DEVICE, "tensor map (pairs)");
        f.qa_spad = spq;
      }
      parse_party_rows(c, f, dq, ncodes, spq, f.qa.as<uint8_t>());
      if (!f.pc.ensure(ncols * ncodes * eb + 16)) return pfail(c, IRISMPC_GPU_ERR_DEVICE, "oom (pair dots)");
      GemmArgs g{};
      g.s_pad = (uint32_t)spq;
      g.nb_rows = ncols_pad;
      g.nkb_seg = c->l_pad / kGemmBK;
      g.nseg = f.nseg;
      g.rep = f.nseg == 2;
      g.nprob = 1;
      g.limbs = L;
      g.s_valid = ncodes;
      g.ncols = (uint32_t)ncols;
      g.out = f.pc.p;
      g.out_pstride = ncols * ncodes;
      g.out_cstride = ncodes;
      launch_gemm(f.tQA, f.tB, g, (uint32_t)(spq / kGemmBM), (uint32_t)cdiv(ncols, bn), st);
      launch_pair_gather(f.pc.p, eb, 1, ncodes, (uint32_t)ncols, persons, r, out + ncols * S * eb, npairs, st);
    }
  }
  PCK(c, cudaGetLastError());
  PCK(c, cudaEventRecord(c->pev[0], st));
  // ---- dot phase: reshare_pair<KH, KM>, own -> next, prev <- previous
  uint32_t* hd_o = c->rs.as<uint32_t>();  // [hd own | ml own | hd prev | ml prev] x (n + 8) u32
  uint32_t* ml_o = hd_o + (n + 8);
  uint32_t* hd_p = hd_o + 2 * (n + 8);
  uint32_t* ml_p = hd_o + 3 * (n + 8);
  const uint64_t msg_bytes = n * (vw.kh / 8) + nml * (vw.km / 8);
  if (!vw.km) {  // plain-mask: no shared ml (the taps read zeros, like the oracle's)
    PCK(c, cudaMemsetAsync(ml_o, 0, (n + 8) * 4, st));
    PCK(c, cudaMemsetAsync(ml_p, 0, (n + 8) * 4, st));
  }
  if (!c->xsend.ensure(msg_bytes + 64) || !c->xrecv.ensure(msg_bytes + 64))
    return pfail(c, IRISMPC_GPU_ERR_DEVICE, "oom (reshare)");
  {
    const unsigned gr = nblk(rup(cdiv(n, 8), 32));
    uint8_t* xs = c->xsend.as<uint8_t>();
    if (vw.kh == 16 && vw.km == 0)
      k_pty_reshare<2, 0><<<gr, kThreads, 0, st>>>(dh, dm, n, c->own, c->prev, c->pos[0], c->pos[1], hd_o, ml_o, xs);
    else if (vw.kh == 16 && vw.km == 16)
      k_pty_reshare<2, 2><<<gr, kThreads, 0, st>>>(dh, dm, n, c->own, c->prev, c->pos[0], c->pos[1], hd_o, ml_o, xs);
    else if (vw.kh == 16)
      k_pty_reshare<2, 4><<<gr, kThreads, 0, st>>>(dh, dm, n, c->own, c->prev, c->pos[0], c->pos[1], hd_o, ml_o, xs);
    else
      k_pty_reshare<4, 4><<<gr, kThreads, 0, st>>>(dh, dm, n, c->own, c->prev, c->pos[0], c->pos[1], hd_o, ml_o, xs);
  }
  PCK(c, cudaGetLastError());
  int rc = step(c, kDot, {{next_of(p), c->xsend.p, msg_bytes}}, {{prev_of(p), c->xrecv.p, msg_bytes}}, {msg_bytes}, 1);
  if (rc) return rc;
  {
    const uint8_t* xr = c->xrecv.as<uint8_t>();
    if (vw.kh == 16 && vw.km == 0)
      k_pty_unpack<2, 0><<<nblk(n), kThreads, 0, st>>>(xr, n, hd_p, ml_p);
    else if (vw.kh == 16 && vw.km == 16)
      k_pty_unpack<2, 2><<<nblk(n), kThreads, 0, st>>>(xr, n, hd_p, ml_p);
    else if (vw.kh == 16)
      k_pty_unpack<2, 4><<<nblk(n), kThreads, 0, st>>>(xr, n, hd_p, ml_p);
    else
      k_pty_unpack<4, 4><<<nblk(n), kThreads, 0, st>>>(xr, n, hd_p, ml_p);
  }
  PCK(c, cudaEventRecord(c->pev[1], st));
  if (!c->rows.ensure(2ull * 32 * W * 8 + 64) || !c->bits.ensure(4ull * W * 8 + 64) ||
      !c->inj.ensure(4ull * (n + 8) * 2 + 64) || !c->ml32.ensure(2 * (n + 8) * 4) || !c->diff.ensure(2 * (n + 8) * 4))
    return pfail(c, IRISMPC_GPU_ERR_DEVICE, "oom (comparison)");
  uint64_t* rows = c->rows.as<uint64_t>();
  uint64_t* b_o = c->bits.as<uint64_t>();  // [inst][W]: bit16, bit17 (mpc-lift)
  uint64_t* b_p = b_o + 2 * W;
  uint32_t* ml32 = c->ml32.as<uint32_t>();  // components laid out [own n+8 | prev n+8]
  uint32_t* diff = c->diff.as<uint32_t>();
  // stream layout: reshare n (+ n), then for mpc-lift the 64 lift
  // gates and the injects (seed 1: 2n, seed 3: 6n), then the MSB gates
  const uint64_t lift_draws[3] = {2 * n, 0, 6 * n};
  uint64_t msb_o = c->pos[0] + n + nml, msb_p = c->pos[1] + n + nml;
  // ---- lane chunks of the comparison phase (lanes are independent until the OR tree)
  static const int env_chunks = [] {
    const char* e = std::getenv("IRISMPC_PARTY_CHUNKS");  // test hook: force 1 or 2
    return e ? std::atoi(e) : 0;
  }();
  const int nch = env_chunks ? std::max(1, std::min(2, env_chunks)) : (W >= 4096 ? 2 : 1);
  std::vector<Chunk> chunks;
  if (nch == 1 || W < 2) {
    chunks.push_back({0, 0, W, 0, n, st});
  } else {
    const uint64_t w1 = W / 2;
    chunks.push_back({0, 0, w1, 0, 64 * w1, c->cs[0]});
    chunks.push_back({1, w1, W - w1, 64 * w1, n - 64 * w1, c->cs[1]});
    PCK(c, cudaEventRecord(c->ej[0], st));
    for (const Chunk& ch : chunks) PCK(c, cudaStreamWaitEvent(ch.st, c->ej[0], 0));
  }
  const int KC = vw.kc;
  if (V == kMpcLift) {
    // ---- lift<16,16>
    uint16_t* i17 = c->inj.as<uint16_t>();  // [comp][n+8]
    uint16_t* i16 = i17 + 2 * (n + 8);
    for (const Chunk& ch : chunks)
      k_pty_split<uint32_t, 16><<<nblk(4 * ch.words), kThreads, 0, ch.st>>>(ml_o + ch.lane0, ml_p + ch.lane0, ch.lanes,
                                                                           W, rows + ch.w0, 2 * ch.words);
    rc = bit_extract(c, kLift, rows, rows + 16 * W, 16, {16, 17}, chunks, n, W, c->pos[0] + 2 * n, c->pos[1] + 2 * n,
                     b_o, b_p);
    if (rc) return rc;
    // seed_1 / seed_3 element bases (own/prev stream positions by role)
    const uint64_t pos1 = p == 0 ? c->pos[0] : (p == 1 ? c->pos[1] : 0);
    const uint64_t pos3 = p == 0 ? c->pos[1] : (p == 2 ? c->pos[0] : 0);
    rc = bit_inject(c, b_o + W, b_p + W, chunks, n, 15, pos1 + 2 * n + 64 * W, pos3 + 2 * n + 64 * W, i17,
                    i17 + n + 8);
    if (rc) return rc;
    rc = bit_inject(c, b_o, b_p, chunks, n, 16, pos1 + 3 * n + 64 * W, pos3 + 5 * n + 64 * W, i16, i16 + n + 8);
    if (rc) return rc;
    for (const Chunk& ch : chunks) {
      const uint64_t L = ch.lane0;
      k_pty_diff<<<nblk(ch.lanes), kThreads, 0, ch.st>>>(ml_o + L, hd_o + L, i17 + L, i16 + L, ch.lanes, c->cfg.a,
                                                         c->cfg.b, ml32 + L, diff + L);
      k_pty_diff<<<nblk(ch.lanes), kThreads, 0, ch.st>>>(ml_p + L, hd_p + L, i17 + n + 8 + L, i16 + n + 8 + L,
                                                         ch.lanes, c->cfg.a, c->cfg.b, ml32 + n + 8 + L,
                                                         diff + n + 8 + L);
    }
    msb_o += 64 * W + lift_draws[ko];
    msb_p += 64 * W + lift_draws[kp];
  } else {
    const int plain = V == kPlainMask;
    const double coef = 1.0 - 2.0 * c->cfg.match_ratio;
    const uint16_t* pub = reinterpret_cast<const uint16_t*>(dm);  // plain-mask: the public popcounts
    for (const Chunk& ch : chunks) {
      const uint64_t L = ch.lane0;
      k_pty_cmp<<<nblk(ch.lanes), kThreads, 0, ch.st>>>(plain, hd_o + L, ml_o + L, pub + L, ch.lanes, c->cfg.a,
                                                        c->cfg.b, coef, p == 0, ml32 + L, diff + L);
      k_pty_cmp<<<nblk(ch.lanes), kThreads, 0, ch.st>>>(plain, hd_p + L, ml_p + L, pub + L, ch.lanes, c->cfg.a,
                                                        c->cfg.b, coef, p == 1, ml32 + n + 8 + L, diff + n + 8 + L);
    }
  }
  PCK(c, cudaGetLastError());
  PCK(c, cudaEventRecord(c->pev[2], chunks[0].st));
  // ---- msb<KC>
  for (const Chunk& ch : chunks) {
    if (KC == 32)
      k_pty_split<uint32_t, 32><<<nblk(4 * ch.words), kThreads, 0, ch.st>>>(
          diff + ch.lane0, diff + n + 8 + ch.lane0, ch.lanes, W, rows + ch.w0, 2 * ch.words);
    else
      k_pty_split<uint32_t, 16><<<nblk(4 * ch.words), kThreads, 0, ch.st>>>(
          diff + ch.lane0, diff + n + 8 + ch.lane0, ch.lanes, W, rows + ch.w0, 2 * ch.words);
  }
  uint64_t* mb_o = b_o + 2 * W;  // msb bit rows (own, prev) in the second half of `bits`
  uint64_t* mb_p = b_o + 3 * W;
  rc = bit_extract(c, kMsb, rows, rows + (uint64_t)KC * W, KC, {KC - 1}, chunks, n, W, msb_o, msb_p, mb_o, mb_p);
  if (rc) return rc;
  if (chunks.size() > 1)
    for (size_t k = 0; k < chunks.size(); ++k) {
      PCK(c, cudaEventRecord(c->ej[1 + k], chunks[k].st));
      PCK(c, cudaStreamWaitEvent(st, c->ej[1 + k], 0));
    }
  PCK(c, cudaEventRecord(c->pev[3], st));
  // ---- taps (parity tests)
  c->tap_n = n;
  // ---- debug rows open to P1
  if (c->cfg.debug_rows && row_bits_out) {
    rc = open_to_p1(c, reinterpret_cast<const uint8_t*>(mb_o), reinterpret_cast<const uint8_t*>(mb_p), n,
                    p == 0 ? row_bits_out : nullptr);
    if (rc) return rc;
  }
  // ---- or_tree_batch (circuits.hpp:387-434): groups of lanes (engine.cpp:262-293)
  std::vector<OrGroup> grp(ngroups);
  std::vector<uint64_t> pair_lanes;
  std::vector<uint64_t> len(ngroups);
  {
    std::vector<std::vector<uint64_t>> pl(ngroups);
    uint64_t k = ncols * S;
    for (uint32_t i = 0; i < persons && !membership; ++i)
      for (uint32_t j = i + 1; j < persons; ++j)
        for (uint32_t e = 0; e < 4 * r; ++e, ++k) {
          pl[i].push_back(k);
          pl[j].push_back(k);
        }
    uint64_t off = 0, woff = 0;
    for (uint32_t g2 = 0; g2 < ngroups; ++g2) {
      OrGroup& G = grp[g2];
      G.db_lane0 = membership ? 0 : (uint64_t)g2 * 2 * r * S;
      G.db_len = membership ? S : 2ull * r * S;
      G.pair_off = off;
      G.len = G.db_len + pl[g2].size();
      G.row_off = woff;
      len[g2] = G.len;
      pair_lanes.insert(pair_lanes.end(), pl[g2].begin(), pl[g2].end());
      off += pl[g2].size();
      woff += cdiv(G.len, 64) + 1;
    }
  }
  uint64_t pool_words = 0, max_w = 0;
  for (auto& G : grp) {
    pool_words += cdiv(G.len, 64) + 1;
    max_w = std::max(max_w, cdiv(G.len, 64));
  }
  if (!c->groups.ensure(ngroups * sizeof(OrGroup) + 16) || !c->pairs.ensure(pair_lanes.size() * 8 + 16) ||
      !c->pool[0].ensure(2 * pool_words * 8 + 16) || !c->pool[1].ensure(2 * pool_words * 8 + 16) ||
      !c->tz[0].ensure(2 * pool_words * 8 + 16) || !c->levels.ensure(ngroups * sizeof(OrLevel) + 16) ||
      !c->rowoff.ensure(ngroups * 8 + 16))
    return pfail(c, IRISMPC_GPU_ERR_DEVICE, "oom (or tree)");
  PCK(c, cudaMemcpyAsync(c->groups.p, grp.data(), ngroups * sizeof(OrGroup), cudaMemcpyHostToDevice, st));
  if (!pair_lanes.empty())
    PCK(c, cudaMemcpyAsync(c->pairs.p, pair_lanes.data(), pair_lanes.size() * 8, cudaMemcpyHostToDevice, st));
  uint64_t* cur[2] = {c->pool[0].as<uint64_t>(), c->pool[0].as<uint64_t>() + pool_words};
  uint64_t* nxt[2] = {c->pool[1].as<uint64_t>(), c->pool[1].as<uint64_t>() + pool_words};
  if (max_w)
    k_pty_or_gather<<<nblk(ngroups * max_w), kThreads, 0, st>>>(c->groups.as<OrGroup>(), ngroups,
                                                                 c->pairs.as<uint64_t>(), mb_o, mb_p, cur[0], cur[1],
                                                                 max_w);
  const uint64_t msb_gates = 2ull * KC - 3;
  const uint64_t or_o = msb_o + msb_gates * W, or_p = msb_p + msb_gates * W;
  std::vector<uint64_t> roff(ngroups);
  for (uint32_t g2 = 0; g2 < ngroups; ++g2) roff[g2] = grp[g2].row_off;
  uint64_t used = 0;
  uint64_t* tzo = c->tz[0].as<uint64_t>();
  uint64_t* tzp = tzo + pool_words;
  for (;;) {
    std::vector<OrLevel> lv;
    uint64_t t_words = 0, counted = 0, max_wb = 0, max_wa = 0;
    for (uint32_t g2 = 0; g2 < ngroups; ++g2) {
      if (len[g2] <= 1) continue;
      OrLevel L{};
      L.src_off = roff[g2];
      L.dst_off = roff[g2];
      L.na = (len[g2] + 1) / 2;
      L.nb = len[g2] - L.na;
      L.wa = cdiv(L.na, 64);
      L.wb = cdiv(L.nb, 64);
      L.t_off = t_words;
      L.eo = or_o + used;
      L.ep = or_p + used;
      used += L.wb;
      t_words += L.wb;
      counted += cdiv(L.nb, 8);
      max_wb = std::max(max_wb, L.wb);
      max_wa = std::max(max_wa, L.wa);
      lv.push_back(L);
      len[g2] = L.na;
    }
    if (lv.empty()) break;
    PCK(c, cudaMemcpyAsync(c->levels.p, lv.data(), lv.size() * sizeof(OrLevel), cudaMemcpyHostToDevice, st));
    k_pty_or_and<<<nblk(lv.size() * max_wb), kThreads, 0, st>>>(c->levels.as<OrLevel>(), (uint32_t)lv.size(), max_wb,
                                                               cur[0], cur[1], c->own, c->prev, tzo);
    rc = step(c, kOr, {{next_of(p), tzo, t_words * 8}}, {{prev_of(p), tzp, t_words * 8}}, {counted}, 1);
    if (rc) return rc;
    k_pty_or_fold<<<nblk(lv.size() * max_wa), kThreads, 0, st>>>(c->levels.as<OrLevel>(), (uint32_t)lv.size(), max_wa,
                                                                cur[0], cur[1], tzo, tzp, nxt[0], nxt[1]);
    // groups that did not fold this round keep their rows: copy them across
    for (uint32_t g2 = 0; g2 < ngroups; ++g2) {
      bool folded = false;
      for (auto& L : lv) folded |= L.src_off == roff[g2];
      if (!folded && grp[g2].len)
        for (int comp = 0; comp < 2; ++comp)
          PCK(c, cudaMemcpyAsync(nxt[comp] + roff[g2], cur[comp] + roff[g2], 8, cudaMemcpyDeviceToDevice, st));
    }
    std::swap(cur[0], nxt[0]);
    std::swap(cur[1], nxt[1]);
    // level table reuse: wait before the next upload overwrites it
    PCK(c, cudaStreamSynchronize(st));
  }
  // ---- open the per-person aggregates at P1
  for (uint32_t g2 = 0; g2 < ngroups; ++g2)
    if (grp[g2].len == 0) roff[g2] = ~0ull;
  PCK(c, cudaMemcpyAsync(c->rowoff.p, roff.data(), ngroups * 8, cudaMemcpyHostToDevice, st));
  if (!c->open_buf[2].ensure(2 * cdiv(ngroups, 8) + 16)) return pfail(c, IRISMPC_GPU_ERR_DEVICE, "oom (open)");
  uint8_t* ob = c->open_buf[2].as<uint8_t>();
  const uint64_t gb = cdiv(ngroups, 8);
  k_pty_pack_groups<<<nblk(gb), kThreads, 0, st>>>(cur[0], c->rowoff.as<uint64_t>(), ngroups, ob);
  k_pty_pack_groups<<<nblk(gb), kThreads, 0, st>>>(cur[1], c->rowoff.as<uint64_t>(), ngroups, ob + gb);
  PCK(c, cudaGetLastError());
  rc = open_to_p1(c, ob, ob + gb, ngroups, p == 0 ? match_out : nullptr);
  if (rc) return rc;
  PCK(c, cudaEventRecord(c->ev[1], st));
  PCK(c, cudaStreamSynchronize(st));
  // ---- stream positions advance exactly as the reference's (A.3)
  const uint64_t glen = membership ? S : 2ull * r * S + (uint64_t)(persons ? persons - 1 : 0) * 4 * r;
  const uint64_t ord = ref_or_draws(ngroups, glen, nullptr);
  c->pos[0] = or_o + ord;
  c->pos[1] = or_p + ord;
  if (stats) {
    std::memset(stats, 0, sizeof(*stats));
    stats->s = S;
    stats->l = c->l;
    stats->batch = membership ? 1 : persons;
    stats->lanes = n;
    stats->dot_bytes = c->led_bytes[kDot];
    stats->lift_bytes = c->led_bytes[kLift] + c->led_bytes[kOt];
    stats->msb_bytes = c->led_bytes[kMsb];
    stats->or_tree_bytes = c->led_bytes[kOr];
    stats->dot_rounds = c->led_rounds[kDot];
    stats->lift_rounds = c->led_rounds[kLift] + c->led_rounds[kOt];
    stats->msb_rounds = c->led_rounds[kMsb];
    stats->or_tree_rounds = c->led_rounds[kOr];
    stats->wire_bytes = c->wire;
    float ms = 0;
    cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]);
    stats->wall_ms = ms;
    const cudaEvent_t b[5] = {c->ev[0], c->pev[0], c->pev[1], c->pev[2], c->pev[3]};
    const cudaEvent_t e[5] = {c->pev[0], c->pev[1], c->pev[2], c->pev[3], c->ev[1]};
    for (int i = 0; i < 5; ++i) {
      cudaEventElapsedTime(&ms, b[i], e[i]);
      stats->phase_ms[i] = ms;
    }
    double xms = 0;  // device time spent inside the transport steps
    for (size_t i = 0; i + 1 < c->nxev; i += 2) {
      cudaEventElapsedTime(&ms, c->xev[i], c->xev[i + 1]);
      xms += ms;
    }
    stats->phase_ms[5] = xms;
  }
  return 0;
}

}  // namespace

// ============================================================== C-ABI

extern "C" {

int irismpc_gpu_nccl_unique_id(uint8_t out[128]) {
  if (!out || !nccl().ok) return IRISMPC_GPU_ERR_DEVICE;
  ncclUniqueId id;
  if (nccl().get_unique_id(&id) != ncclSuccess) return IRISMPC_GPU_ERR_DEVICE;
  std::memcpy(out, &id, 128);
  return 0;
}

int irismpc_gpu_party_create_nccl(const irismpc_gpu_config* cfg, uint32_t party, const uint8_t nccl_id[128],
                                  irismpc_gpu_party** out) {
  std::string why;
  int rc = party_init(cfg, party, out, &why);
  if (rc) {
    if (!why.empty()) std::fprintf(stderr, "irismpc_gpu_party_create: %s\n", why.c_str());
    return rc;
  }
  if (!nccl().ok) {
    irismpc_gpu_party_destroy(*out);
    *out = nullptr;
    return IRISMPC_GPU_ERR_DEVICE;
  }
  auto* t = new NcclTransport;
  ncclUniqueId id;
  std::memcpy(&id, nccl_id, 128);
  if (nccl().comm_init_rank(&t->comm, 3, id, (int)party - 1) != ncclSuccess) {
    delete t;
    irismpc_gpu_party_destroy(*out);
    *out = nullptr;
    return IRISMPC_GPU_ERR_DEVICE;
  }
  (*out)->net = t;
  return 0;
}

int irismpc_gpu_inproc_create(irismpc_gpu_inproc** out) {
  if (!out) return IRISMPC_GPU_ERR_CONFIG;
  *out = new irismpc_gpu_inproc;
  return 0;
}

void irismpc_gpu_inproc_destroy(irismpc_gpu_inproc* net) {
  if (!net) return;
  for (auto& row : net->q)
    for (auto& q : row)
      for (auto& it : q) {
        cudaFree(it.buf);
        cudaEventDestroy(it.ev);
      }
  delete net;
}

int irismpc_gpu_party_create_inproc(const irismpc_gpu_config* cfg, uint32_t party, irismpc_gpu_inproc* net,
                                    irismpc_gpu_party** out) {
  if (!net) return IRISMPC_GPU_ERR_CONFIG;
  std::string why;
  int rc = party_init(cfg, party, out, &why);
  if (rc) {
    if (!why.empty()) std::fprintf(stderr, "irismpc_gpu_party_create: %s\n", why.c_str());
    return rc;
  }
  auto* t = new InProcTransport;
  t->net = net;
  (*out)->net = t;
  return 0;
}

void irismpc_gpu_party_destroy(irismpc_gpu_party* c) {
  if (!c) return;
  cudaSetDevice(c->cfg.device);
  cudaStreamSynchronize(c->st);
  DBuf* bufs[] = {&c->qpay, &c->dots, &c->rs, &c->rows, &c->carry, &c->chain, &c->zbuf, &c->zrecv, &c->inj,
                  &c->msg, &c->msg2, &c->ml32, &c->diff, &c->bits, &c->pairs, &c->groups, &c->levels, &c->pool[0],
                  &c->pool[1], &c->tz[0], &c->tz[1], &c->rowoff, &c->open_buf[0], &c->open_buf[1], &c->open_buf[2],
                  &c->xsend, &c->xrecv, &c->c2buf};
  for (DBuf* b : bufs) b->release();
  for (auto& f : c->fld) {
    f.db.release();
    f.q.release();
    f.qa.release();
    f.pc.release();
  }
  delete c->net;
  cudaEventDestroy(c->ev[0]);
  cudaEventDestroy(c->ev[1]);
  for (auto& e : c->pev) cudaEventDestroy(e);
  for (auto& e : c->xev) cudaEventDestroy(e);
  for (auto& e : c->ea) cudaEventDestroy(e);
  for (auto& e : c->eb) cudaEventDestroy(e);
  for (auto& e : c->ej) cudaEventDestroy(e);
  cudaStreamSynchronize(c->cst);
  for (auto& x : c->cs) {
    cudaStreamSynchronize(x);
    cudaStreamDestroy(x);
  }
  cudaStreamDestroy(c->cst);
  cudaStreamDestroy(c->st);
  delete c;
}

const char* irismpc_gpu_party_last_error(const irismpc_gpu_party* c) { return c ? c->err.c_str() : "null context"; }

int irismpc_gpu_party_load_db(irismpc_gpu_party* c, const uint8_t* payload, size_t len, uint64_t s) {
  if (!c) return IRISMPC_GPU_ERR_CONFIG;
  cudaSetDevice(c->cfg.device);
  if (len != s * c->rec) return pfail(c, IRISMPC_GPU_ERR_CONFIG, "db payload size mismatch");
  c->db_loaded = false;
  c->s = s;
  c->s_pad = rup(s ? s : 1, 2 * kGemmBM);
  DBuf stage;
  if (!stage.ensure(len)) return pfail(c, IRISMPC_GPU_ERR_DEVICE, "oom (db staging)");
  PCK(c, cudaMemcpyAsync(stage.p, payload, len, cudaMemcpyHostToDevice, c->st));
  for (auto& f : c->fld) {
    const uint64_t rows = (uint64_t)f.slots * f.fmt.limbs * c->s_pad;
    if (!f.db.ensure(rows * c->l_pad)) return pfail(c, IRISMPC_GPU_ERR_DEVICE, "oom (db planes)");
    PCK(c, cudaMemsetAsync(f.db.p, 0, rows * c->l_pad, c->st));
    if (make_plane_tmap(&f.tA, f.db.p, rows, c->l_pad, kGemmBM))
      return pfail(c, IRISMPC_GPU_ERR_DEVICE, "tensor map (db)");
    parse_party_rows(c, f, stage.as<uint8_t>(), s, c->s_pad, f.db.as<uint8_t>());
  }
  PCK(c, cudaGetLastError());
  PCK(c, cudaStreamSynchronize(c->st));
  stage.release();
  c->db_loaded = true;
  return 0;
}

int irismpc_gpu_party_batch_query(irismpc_gpu_party* c, const uint8_t* q, size_t qlen, uint32_t persons,
                                  uint8_t* person_match_out, uint8_t* row_bits_out, irismpc_gpu_party_stats* stats) {
  if (!c) return IRISMPC_GPU_ERR_CONFIG;
  cudaSetDevice(c->cfg.device);
  return party_query(c, q, qlen, persons, 0, person_match_out, row_bits_out, stats);
}

int irismpc_gpu_party_membership(irismpc_gpu_party* c, const uint8_t* q, size_t qlen, uint8_t* match_out,
                                 uint8_t* row_bits_out, irismpc_gpu_party_stats* stats) {
  if (!c) return IRISMPC_GPU_ERR_CONFIG;
  cudaSetDevice(c->cfg.device);
  return party_query(c, q, qlen, 1, 1, match_out, row_bits_out, stats);
}

int irismpc_gpu_party_read_tap(irismpc_gpu_party* c, int tap, void* host_out, size_t bytes) {
  if (!c || !host_out) return IRISMPC_GPU_ERR_CONFIG;
  cudaSetDevice(c->cfg.device);
  const uint64_t n = c->tap_n, W = cdiv(n, 64);
  std::vector<uint8_t> tmp;
  auto copy2 = [&](const void* a, const void* b, size_t esz) -> int {  // [own n][prev n]
    if (bytes < 2 * n * esz) return pfail(c, IRISMPC_GPU_ERR_CONFIG, "tap buffer too small");
    PCK(c, cudaMemcpy(host_out, a, n * esz, cudaMemcpyDeviceToHost));
    PCK(c, cudaMemcpy(static_cast<uint8_t*>(host_out) + n * esz, b, n * esz, cudaMemcpyDeviceToHost));
    return 0;
  };
  switch (tap) {
    case IRISMPC_GPU_TAP_DOT_HD:
    case IRISMPC_GPU_TAP_DOT_ML: {
      const int fi = tap == IRISMPC_GPU_TAP_DOT_ML ? 1 : 0;
      const int hbb = c->fld[0].fmt.limbs == 4 ? 4 : 2, eb = c->fld[fi].fmt.limbs == 4 ? 4 : 2;
      if (bytes < n * eb) return pfail(c, IRISMPC_GPU_ERR_CONFIG, "tap buffer too small");
      const uint8_t* d = c->dots.as<uint8_t>() + (fi ? rup((n + 8) * hbb, 16) : 0);
      PCK(c, cudaMemcpy(host_out, d, n * eb, cudaMemcpyDeviceToHost));
      return 0;
    }
    case IRISMPC_GPU_TAP_RS_HD:
      return copy2(c->rs.as<uint32_t>(), c->rs.as<uint32_t>() + 2 * (n + 8), 4);
    case IRISMPC_GPU_TAP_RS_ML:
      return copy2(c->rs.as<uint32_t>() + n + 8, c->rs.as<uint32_t>() + 3 * (n + 8), 4);
    case IRISMPC_GPU_TAP_ML32:
      return copy2(c->ml32.as<uint32_t>(), c->ml32.as<uint32_t>() + n + 8, 4);
    case IRISMPC_GPU_TAP_DIFF:
      return copy2(c->diff.as<uint32_t>(), c->diff.as<uint32_t>() + n + 8, 4);
    case IRISMPC_GPU_TAP_MSB: {
      if (bytes < 2 * n) return pfail(c, IRISMPC_GPU_ERR_CONFIG, "tap buffer too small");
      std::vector<uint64_t> w(2 * W);
      PCK(c, cudaMemcpy(w.data(), c->bits.as<uint64_t>() + 2 * W, 2 * W * 8, cudaMemcpyDeviceToHost));
      uint8_t* o = static_cast<uint8_t*>(host_out);
      for (int comp = 0; comp < 2; ++comp)
        for (uint64_t i = 0; i < n; ++i) o[comp * n + i] = (uint8_t)((w[comp * W + i / 64] >> (i % 64)) & 1);
      return 0;
    }
    default:
      return pfail(c, IRISMPC_GPU_ERR_CONFIG, "unknown tap");
  }
}

int irismpc_gpu_party_stream_positions(const irismpc_gpu_party* c, uint64_t pos[2]) {
  if (!c || !pos) return IRISMPC_GPU_ERR_CONFIG;
  pos[0] = c->pos[0];
  pos[1] = c->pos[1];
  return 0;
}

}  // extern "C"
