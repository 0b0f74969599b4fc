// C-ABI of the B200 irismpc hot path (include/irismpc_gpu.h).
//
// One context = the three parties of one DB shard on one GPU.  A query runs
//   K1 parse/rotate query -> (pairs) -> per column chunk: K2 limb GEMM ->
//   K4 threshold (+ fused first OR level) -> K5 per-person OR -> open at P1
// on a single CUDA stream.  Mirrors Session::load_db / batch_query /
// membership (/root/reference/proj/src/engine.cpp:136-398).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <condition_variable>
#include <cstdio>
#include <memory>
#include <mutex>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/irismpc_gpu.h"
#include "common.cuh"
#include "kernels.h"
#include "nccl_api.h"

using namespace irisgpu;

namespace {

struct Buf {
  void* p = nullptr;
  size_t cap = 0;
  int ensure(size_t bytes) {
    if (bytes <= cap && p) return 0;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    if (cudaMalloc(&p, bytes ? bytes : 16) != cudaSuccess) return -1;
    cap = bytes ? bytes : 16;
    return 0;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
  template <class T>
  T* as() const { return static_cast<T*>(p); }
};

uint64_t ceil_div(uint64_t a, uint64_t b) { return (a + b - 1) / b; }

// NVTX range over a C-ABI call (host timeline in nsys / ncu; no-op without a tool)
struct Range {
  explicit Range(const char* name) { nvtxRangePushA(name); }
  ~Range() { nvtxRangePop(); }
};
uint64_t round_up(uint64_t a, uint64_t b) { return ceil_div(a, b) * b; }

// ---- host-side ChaCha / seeds / lambda (setup only) ------------------------
void host_block(const uint8_t seed[16], uint64_t block, uint64_t stream, uint32_t out[16]) {
  SeedKey k;
  std::memcpy(k.k, seed, 16);
  chacha12_block(k, block, stream, out);
}
void host_derive(const uint8_t parent[16], uint64_t tag, uint8_t out[16]) {
  uint32_t blk[16];
  host_block(parent, tag, 0xD5A1u, blk);  // CtrPrf::derive (prf.hpp:106-112)
  std::memcpy(out, blk, 16);
}
void host_seed_from_u64(uint64_t v, uint8_t out[16]) {
  uint8_t s[16] = {0};
  std::memcpy(s, &v, 8);
  host_derive(s, 0, out);
}
SeedKey key_of(const uint8_t* seed) {
  SeedKey k;
  std::memcpy(k.k, seed, 16);
  return k;
}

// party_lagrange_at_zero<32> over {1, X, 1+X} (galois.hpp:66-128); the 16-bit
// lambdas are its low halves (the same closed forms 1+2X, -(1+2X), 1)
struct Gr {
  uint32_t c0, c1;
};
Gr gmul(Gr a, Gr b) {
  return {a.c0 * b.c0 + a.c1 * b.c1, a.c0 * b.c1 + a.c1 * b.c0 + a.c1 * b.c1};
}
Gr gsub(Gr a, Gr b) { return {a.c0 - b.c0, a.c1 - b.c1}; }
Gr ginv(Gr a) {
  Gr y = (a.c1 & 1) == 0 ? Gr{1, 0} : ((a.c0 & 1) == 0 ? Gr{1, 1} : Gr{0, 1});
  for (unsigned c = 1; c < 32; c *= 2) y = gmul(y, gsub(Gr{2, 0}, gmul(a, y)));
  return y;
}
void lambdas(uint32_t out[6]) {
  const Gr xs[3] = {{1, 0}, {0, 1}, {1, 1}};
  for (int i = 0; i < 3; ++i) {
    Gr num{1, 0}, den{1, 0};
    for (int j = 0; j < 3; ++j) {
      if (j == i) continue;
      num = gmul(num, xs[j]);
      den = gmul(den, gsub(xs[j], xs[i]));
    }
    const Gr l = gmul(num, ginv(den));
    out[2 * i] = l.c0;
    out[2 * i + 1] = l.c1;
  }
}

// code_record_bytes / mask_record_bytes (shares.cpp:49-59)
uint64_t field_bytes(uint32_t backend, int bits, uint32_t l) {
  if (bits == 0) return l / 8;
  return backend == IRISMPC_GPU_BACKEND_REPLICATED ? (uint64_t)l * 2 * (bits / 8) : (uint64_t)l * (bits / 8);
}
size_t record_bytes(uint32_t backend, uint32_t variant, uint32_t l) {
  const VariantWidths w = variant_widths((int)variant);
  return field_bytes(backend, w.kh, l) + field_bytes(backend, w.km, l);
}

// Reference or_tree_batch zero_word draws for `groups` equal groups of `len`
// lanes (circuits.hpp:394-427): keeps the seed streams in lockstep with the
// reference across queries on a persistent context.
uint64_t ref_or_draws(uint64_t groups, uint64_t len, uint64_t* rounds, uint64_t* bytes) {
  uint64_t draws = 0, r = 0, b = 0;
  while (len > 1) {
    const uint64_t na = (len + 1) / 2, nb = len - na;
    draws += groups * ceil_div(nb, 64);
    b += groups * ceil_div(nb, 8);
    len = na;
    ++r;
  }
  if (rounds) *rounds = r;
  if (bytes) *bytes = b;
  return draws;
}

}  // namespace

// ---- DB-sharded queries: the two exchanges of SURVEY §8e -------------------
// (1) broadcast of the three query payloads from shard 0, (2) gather of every
// shard's per-person XOR-shared OR partials to shard 0.  Over NCCL (one process
// or thread per GPU) or an in-process group (several contexts in one process,
// e.g. on one GPU, which one NCCL communicator cannot hold).
namespace {

struct ShardComm {
  uint32_t world = 1, rank = 0;
  virtual ~ShardComm() = default;
  virtual std::string bcast(void* dev, size_t bytes, cudaStream_t st) = 0;  // in place, root 0
  // every shard's `bytes` of send -> root's recv[world][bytes] (other ranks' recv may be unused)
  virtual std::string gather(const void* send, void* recv, size_t bytes, cudaStream_t st) = 0;
};

struct NcclShardComm : ShardComm {
  ncclComm_t comm = nullptr;
  // a second communicator (ncclCommSplit of the first) for the streaming path's gathers on
  // the threshold stream while the next query's broadcast runs on the GEMM stream: NCCL
  // operations of one communicator must not be in flight on two streams at once
  ncclComm_t comm2 = nullptr;
  ~NcclShardComm() override {
    if (comm2 && nccl().ok) nccl().comm_destroy(comm2);
    if (comm && nccl().ok) nccl().comm_destroy(comm);
  }
  std::string bcast(void* dev, size_t bytes, cudaStream_t st) override {
    if (!bytes) return "";
    const ncclResult_t r = nccl().broadcast(dev, dev, bytes, ncclUint8, 0, comm, st);
    return r == ncclSuccess ? "" : std::string("nccl broadcast: ") + nccl().error_string(r);
  }
  std::string gather(const void* send, void* recv, size_t bytes, cudaStream_t st) override {
    const ncclResult_t r = nccl().all_gather(send, recv, bytes, ncclUint8, comm, st);
    return r == ncclSuccess ? "" : std::string("nccl all_gather: ") + nccl().error_string(r);
  }
};

}  // namespace

// In-process shard group: a generation barrier plus device copies (cudaMemcpy
// with UVA; peer devices or the same device).
struct irismpc_gpu_shard_group {
  uint32_t world = 1;
  std::mutex mu;
  std::condition_variable cv;
  uint32_t arrived = 0;
  uint64_t gen = 0;
  std::vector<const void*> ptr;
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const uint64_t g = gen;
    if (++arrived == world) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

namespace {

struct InprocShardComm : ShardComm {
  irismpc_gpu_shard_group* g = nullptr;
  std::string bcast(void* dev, size_t bytes, cudaStream_t st) override {
    if (cudaStreamSynchronize(st) != cudaSuccess) return "shard bcast: device fault";
    if (rank == 0) g->ptr[0] = dev;
    g->barrier();
    std::string err;
    if (rank != 0 && bytes &&
        (cudaMemcpyAsync(dev, g->ptr[0], bytes, cudaMemcpyDefault, st) != cudaSuccess ||
         cudaStreamSynchronize(st) != cudaSuccess))
      err = "shard bcast: copy failed";
    g->barrier();  // the root's buffer stays untouched until every shard copied it
    return err;
  }
  std::string gather(const void* send, void* recv, size_t bytes, cudaStream_t st) override {
    if (cudaStreamSynchronize(st) != cudaSuccess) return "shard gather: device fault";
    g->ptr[rank] = send;
    g->barrier();
    std::string err;
    if (rank == 0)
      for (uint32_t r = 0; r < world && err.empty(); ++r)
        if (cudaMemcpyAsync(static_cast<uint8_t*>(recv) + r * bytes, g->ptr[r], bytes, cudaMemcpyDefault, st) !=
                cudaSuccess ||
            cudaStreamSynchronize(st) != cudaSuccess)
          err = "shard gather: copy failed";
    g->barrier();
    return err;
  }
};

}  // namespace

// Device planes of one record field (code -> hd, mask -> ml): DB limb planes
// (A), rotated query planes (B), the unrotated query planes of the pair GEMM
// (A) and its output.
struct FieldPlanes {
  FieldFmt fmt{};
  uint32_t nparty = 3;  // 3 share planes, or 1 public bit plane
  uint32_t nseg = 1;    // 2 for replicated shares ([x_p | x_{p-1}])
  int out_bytes = 2;    // GEMM output element: u16, or u32 for 4 limbs
  Buf db, q, qa, pair_c;
  CUtensorMap tA, tB, tQA;
  uint32_t ncols_pad_cur = 0;
  uint64_t qa_spad = 0;
  // rotation-pair GEMM (prep.cu): S = E + O planes of the DB, D0 / M / D1 query planes
  Buf sdb, rpq;
  CUtensorMap tS, tRP;
  bool rpg = false;  // S planes resident: rotated queries run the RP GEMMs
  bool rpc = false;  // S planes built per row chunk into sch (DB too large for resident S)
  bool rpconv = false;  // ... or formed in the GEMM's shared memory from E and O (GemmArgs::s_conv)
  Buf sch;
  CUtensorMap tSc;
  uint64_t sch_spad = 0;
  uint32_t rp_ncols_cur = 0;
  uint32_t bn() const { return gemm_bn((uint32_t)fmt.limbs); }
  void release() {
    db.release();
    q.release();
    qa.release();
    pair_c.release();
    sdb.release();
    rpq.release();
    sch.release();
    rpg = false;
    rpc = false;
    rpconv = false;
    sch_spad = 0;
    rp_ncols_cur = 0;
    ncols_pad_cur = 0;
    qa_spad = 0;
  }
};

// One in-flight batch query's buffers (irismpc_gpu_batch_query_submit): the
// GEMM stream (st) runs ahead into the next query while the threshold stream
// (st2) finishes this one, so everything the threshold side of a query reads
// after its prep -- segment table, OR slot ranges, pair dots, match words --
// and its result buffers are per slot; two slots alternate.
struct QSlot {
  Buf segs, slot_begin, match[3], pair_dots, open_out;
  Buf qpay[3], part, all;  // streaming sharded queries: broadcast payloads, own / gathered partials
  Seg* h_segs = nullptr;
  size_t h_segs_cap = 0;
  uint8_t* h_match = nullptr;  // pinned copy of the opened person bits
  size_t h_match_cap = 0;
  cudaEvent_t ev[6] = {};
  cudaEvent_t done = nullptr;
  std::vector<cudaEvent_t> gev;  // per chunk: GEMM start / stop
  bool inflight = false;
  uint64_t ticket = 0;
  // what finish_slot needs
  int mode = 0;
  uint32_t ngroups = 0;
  uint8_t* match_out = nullptr;
  uint8_t* row_bits_out = nullptr;
  uint64_t n = 0, nchunks = 0;
  irismpc_gpu_stats stats{};
  bool want_stats = false;
};

struct irismpc_gpu_ctx {
  irismpc_gpu_config cfg{};
  std::string err;
  cudaStream_t st = nullptr, st2 = nullptr, st3 = nullptr;  // GEMM / threshold front / threshold back
  int shamir = 0;
  int variant = kMpcLift;
  VariantWidths vw{16, 16, 32};
  uint32_t l = 0, l_pad = 0;
  uint64_t rec = 0;
  SeedKey keys[3];
  // DB shard
  uint64_t s = 0, s_pad = 0;
  bool db_loaded = false;
  FieldPlanes fld[2];  // 0 code, 1 mask
  // query scratch
  Buf q_pay[3];
  Buf dots, pair_dots, segs, partial, slot_begin, person_out, match[3], open_out;
  Buf ml_rs, diff, gate, bits;  // comparison-only work buffers
  Buf or_scr[2];                // OR-tree level rows (ping-pong)
  uint32_t last_groups = 0;     // groups of the last OR (person_out = [3][last_groups])
  // batch-query threshold work buffers, two sets: job k's front half (keystream,
  // reshare on st2) runs while job k-1's back half (lift, inject, msb on st3) does
  Buf wk_ml_rs[2], wk_diff[2], wk_gate[2], wk_bits[2];
  cudaEvent_t front_done[2] = {nullptr, nullptr}, back_done[2] = {nullptr, nullptr};
  uint64_t job_ctr = 0;
  std::vector<Seg> h_segs;
  Seg* h_segs_pinned = nullptr;
  size_t h_segs_cap = 0;
  // PRF stream state
  uint64_t pos[3] = {0, 0, 0};
  uint64_t query_id = 0;  // queries run on this context (64-bit: never wraps)
  uint64_t or_ctr = 0;    // OR-gate stream counter of the last query (or_stream_id)
  // taps
  bool taps = false;
  bool serial = false;  // irismpc_gpu_profile: one stream, per-kernel CUDA events
  int thr_tile = 0;     // irismpc_gpu_threshold_kernels: the tile reshare / inject kernels in batch queries
  // row-sampled L1 taps (irismpc_gpu_tap_rows): DOT_HD / DOT_ML of these local rows, all columns
  Buf tap_rows_dev;
  uint32_t tap_k = 0;
  Buf tap_buf[7];
  size_t tap_bytes[7] = {0, 0, 0, 0, 0, 0, 0};
  uint64_t tap_n = 0;
  cudaEvent_t ev[6];
  std::unique_ptr<ShardComm> shard;  // DB-sharded queries (irismpc_gpu_shard_attach_*)
  NcclShardComm* shard_nccl = nullptr;  // the same object when attached over NCCL (streaming)
  Buf shard_part, shard_all;
  std::vector<cudaEvent_t> evg, evt;  // chunk pipeline: GEMM done (st); evt[0]: last back half done (st3)
  QSlot qs[2];
  int par = 0;                 // slot of the next query
  uint64_t tickets = 0;        // submitted batch queries
  uint64_t chunk_ctr = 0;      // dot buffer of the next row chunk (continues across queries)
  static constexpr int kMaxDotBufs = 4;
  cudaEvent_t half_free[kMaxDotBufs] = {};  // threshold of the last chunk that read each dot buffer
};

namespace {

int fail(irismpc_gpu_ctx* c, int code, const std::string& msg) {
  if (c) c->err = msg;
  return code;
}

#define CK(ctx, x)                                                                      \
  do {                                                                                  \
    cudaError_t e_ = (x);                                                               \
    if (e_ != cudaSuccess)                                                              \
      return fail(ctx, IRISMPC_GPU_ERR_DEVICE, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

int validate(const irismpc_gpu_config* c, std::string* why) {
  // EngineConfig::validate (engine.cpp:21-34)
  if (c->variant > IRISMPC_GPU_VARIANT_NO_LIFT) {
    *why = "unknown variant";
    return IRISMPC_GPU_ERR_CONFIG;
  }
  if (c->backend > 1) {
    *why = "unknown backend";
    return IRISMPC_GPU_ERR_CONFIG;
  }
  if (c->l == 0 || c->l % 8 != 0) {
    *why = "l must be a positive multiple of 8";
    return IRISMPC_GPU_ERR_BOUNDS;
  }
  if (c->a > c->b) {
    *why = "threshold numerator exceeds denominator";
    return IRISMPC_GPU_ERR_BOUNDS;
  }
  if (c->variant == IRISMPC_GPU_VARIANT_PLAIN_MASK) {
    // check_public_mask_bound(l, 16) (iris.hpp:189-194, 207-211)
    const uint64_t t = 1ull << 16;
    if (!(c->l < t / 4 && c->l < t - (t >> 1))) {
      *why = "comparison ring too small for vector length (public masks)";
      return IRISMPC_GPU_ERR_BOUNDS;
    }
  } else {
    if (c->m != 16 || c->b != (1u << 16)) {
      *why = "shared-mask variants fix b = 2^16";
      return IRISMPC_GPU_ERR_BOUNDS;
    }
    const uint64_t t = 1ull << 32, bl = (uint64_t)c->b * c->l;
    if (!(bl < t / 4 && bl < t - (t >> 1))) {
      *why = "comparison ring too small for b*l (shared masks)";
      return IRISMPC_GPU_ERR_BOUNDS;
    }
  }
  if (c->rotations % 2 == 0) {
    *why = "rotations must be odd";
    return IRISMPC_GPU_ERR_BOUNDS;
  }
  if (c->rotations > 31) {
    *why = "the GPU path supports at most 31 rotations";
    return IRISMPC_GPU_ERR_CONFIG;
  }
  if (c->backend == IRISMPC_GPU_BACKEND_SHAMIR && c->rotations > 1 && (c->l / 64) % 2 != 0) {
    *why = "shamir packing needs an even rotation stride (l/64)";
    return IRISMPC_GPU_ERR_BOUNDS;
  }
  return 0;
}

uint64_t s_total(const irismpc_gpu_ctx* c) {
  return c->cfg.db_rows_total ? c->cfg.db_rows_total : c->s;
}

int drain(irismpc_gpu_ctx* c);

int alloc_planes(irismpc_gpu_ctx* c, uint64_t s) {
  if (int rc = drain(c)) return rc;
  for (auto& f : c->fld) {
    f.db.release();
    f.sdb.release();
    f.rpg = false;
  }
  c->db_loaded = false;
  c->s = s;
  c->s_pad = round_up(s ? s : 1, 2 * kGemmBM);  // CTA-pair tiles cover 256 rows
  for (auto& f : c->fld) {
    const uint64_t rows = (uint64_t)f.nparty * f.fmt.limbs * c->s_pad;
    const size_t bytes = rows * c->l_pad;
    if (f.db.ensure(bytes)) return fail(c, IRISMPC_GPU_ERR_DEVICE, "out of device memory for the DB planes");
    CK(c, cudaMemsetAsync(f.db.p, 0, bytes, c->st));
    if (make_plane_tmap(&f.tA, f.db.p, rows, c->l_pad, kGemmBM))
      return fail(c, IRISMPC_GPU_ERR_DEVICE, "cuTensorMapEncodeTiled failed for the DB planes");
  }
  return 0;
}

// parse `rows` rows (device payloads) into planes at row0
int parse_rows(irismpc_gpu_ctx* c, const uint8_t* const dp[3], uint64_t rows, uint64_t row0, Buf* bad) {
  for (auto& f : c->fld) {
    if (!c->shamir && bad) launch_check_rep(dp[0], dp[1], dp[2], rows, f.fmt, c->l, bad->as<int>(), c->st);
    for (uint32_t p = 0; p < f.nparty; ++p)
      launch_parse_field(dp[p], rows, row0, c->l, c->l_pad, c->s_pad, (int)p, c->shamir, f.fmt, f.db.as<uint8_t>(),
                         c->st);
  }
  CK(c, cudaGetLastError());
  return 0;
}

int finish_load(irismpc_gpu_ctx* c, Buf* bad) {
  if (bad) {
    int h = 0;
    CK(c, cudaMemcpyAsync(&h, bad->p, sizeof(int), cudaMemcpyDeviceToHost, c->st));
    CK(c, cudaStreamSynchronize(c->st));
    if (h) return fail(c, IRISMPC_GPU_ERR_INCONSISTENT, "replicated share cross-check failed at load");
  }
  // RP: S = E + O planes (1.5x the DB planes in all).  A DB too large for them keeps the
  // plain GEMM on the same (permuted) planes.
  static const bool rp_layout_only = [] {
    const char* e = std::getenv("IRISMPC_RP");
    return e && std::string(e) == "layout";
  }();
  // opt-in: per-chunk S planes when resident ones do not fit ("force": always, tests);
  // "conv" / "conv_force": S = E + O formed inside the GEMM instead (no S planes at all)
  static const int rp_chunked = [] {
    const char* e = std::getenv("IRISMPC_RP_CHUNKED");
    if (!e || std::string(e) == "0") return 0;
    const std::string v(e);
    return v == "force" ? 2 : v == "conv" ? 3 : v == "conv_force" ? 4 : 1;
  }();
  for (auto& f : c->fld) {
    f.rpg = false;
    f.rpc = false;
    f.rpconv = false;
    if (!f.fmt.rp || rp_layout_only) continue;
    f.rpc = rp_chunked != 0;
    f.rpconv = rp_chunked >= 3;
    if (rp_chunked == 2 || rp_chunked == 4) continue;
    const uint64_t rows = (uint64_t)f.nparty * f.fmt.limbs * c->s_pad;
    // keep 16 GB free for the query's work buffers (dots, gate keystream, planes)
    size_t free_b = 0, total_b = 0;
    if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess || free_b < rows * (c->l / 2) + (16ull << 30)) continue;
    if (f.sdb.ensure(rows * (c->l / 2))) {
      cudaGetLastError();  // out of memory is not sticky: clear it and run without RP
      continue;
    }
    launch_rp_sum(f.db.as<uint8_t>(), f.nparty, c->s_pad, c->l, c->l_pad, f.fmt.limbs, f.sdb.as<uint8_t>(), c->st);
    CK(c, cudaGetLastError());
    if (make_plane_tmap(&f.tS, f.sdb.p, rows, c->l / 2, kGemmBM))
      return fail(c, IRISMPC_GPU_ERR_DEVICE, "cuTensorMapEncodeTiled failed for the RP sum planes");
    f.rpg = true;
    f.rpc = false;
    f.rpconv = false;
  }
  CK(c, cudaStreamSynchronize(c->st));
  c->db_loaded = true;
  return 0;
}

int ensure_query_buffers(irismpc_gpu_ctx* c, uint32_t ncols_pad) {
  for (auto& f : c->fld) {
    const uint64_t rows = (uint64_t)f.nparty * f.nseg * f.fmt.limbs * ncols_pad;
    const size_t bytes = rows * c->l_pad;
    if (bytes > f.q.cap || ncols_pad != f.ncols_pad_cur) {
      if (f.q.ensure(bytes)) return fail(c, IRISMPC_GPU_ERR_DEVICE, "out of device memory for query planes");
      CK(c, cudaMemsetAsync(f.q.p, 0, bytes, c->st));
      if (make_plane_tmap(&f.tB, f.q.p, rows, c->l_pad, f.bn() / 2))
        return fail(c, IRISMPC_GPU_ERR_DEVICE, "cuTensorMapEncodeTiled failed for the query planes");
      f.ncols_pad_cur = ncols_pad;
    }
  }
  return 0;
}

int ensure_host_segs(irismpc_gpu_ctx* c, size_t n) {
  if (n <= c->h_segs_cap) return 0;
  if (c->h_segs_pinned) cudaFreeHost(c->h_segs_pinned);
  c->h_segs_pinned = nullptr;
  CK(c, cudaMallocHost(&c->h_segs_pinned, n * sizeof(Seg)));
  c->h_segs_cap = n;
  return 0;
}

GemmArgs field_gemm_args(const irismpc_gpu_ctx* c, const FieldPlanes& f, uint32_t ncols_pad) {
  GemmArgs g{};
  g.nb_rows = ncols_pad;
  g.nkb_seg = c->l_pad / kGemmBK;
  g.nseg = f.nseg;
  g.rep = f.nseg == 2 ? 1 : 0;
  g.nprob = f.nparty;
  g.limbs = (uint32_t)f.fmt.limbs;
  return g;
}

// Core query on device payloads.  mode 0: final (open into match_out host),
// 1: partial (component bits into partial_dev).
//
// DB lanes run in row chunks: K2 GEMMs (code field, mask field) of chunk i on
// stream st while the K4 threshold pipeline of chunk i-1 runs on stream st2
// (tensor pipe vs ALU pipes), dot outputs double-buffered.  The pair lanes,
// the per-person OR and the open follow on st2 / st.
int finish_slot(irismpc_gpu_ctx* c, QSlot& q);

int run_query(irismpc_gpu_ctx* c, const uint8_t* const dq[3], const size_t qlen[3], uint32_t persons,
              int membership, int mode, uint8_t* match_out, uint8_t* row_bits_out, uint8_t* partial_dev,
              irismpc_gpu_stats* stats, bool host_input, const uint8_t* const hq[3], uint64_t* ticket_out = nullptr) {
  if (!c->db_loaded) return fail(c, IRISMPC_GPU_ERR_CONFIG, "no database loaded");
  // the slot this query uses: its previous occupant (two queries back) must be done
  QSlot& Q = c->qs[c->par];
  if (Q.inflight) {
    const int rc = finish_slot(c, Q);
    if (rc) return rc;
  }
  const size_t rec = c->rec;
  const uint32_t ncodes = membership ? 1u : 2u * persons;
  for (int p = 0; p < 3; ++p) {
    if (qlen[p] % rec != 0) return fail(c, IRISMPC_GPU_ERR_CONFIG, "query payload size mismatch");
    if (qlen[p] / rec != ncodes)
      return fail(c, IRISMPC_GPU_ERR_CONFIG,
                  membership ? "membership expects exactly one query code"
                             : "batch query expects 2 codes per person");
  }
  const int V = c->variant;
  const VariantWidths vw = c->vw;
  const bool shared_ml = vw.km != 0;
  FieldPlanes& fh = c->fld[0];
  FieldPlanes& fm = c->fld[1];
  const uint64_t hb = (uint64_t)fh.out_bytes, mb = (uint64_t)fm.out_bytes;  // dot element bytes
  const uint32_t r = membership ? 1u : c->cfg.rotations;
  const uint64_t ncols = (uint64_t)ncodes * r;
  const uint32_t ncols_pad = (uint32_t)round_up(ncols ? ncols : 1, kGemmBN);
  const uint64_t S = s_total(c);
  const bool rank0 = c->cfg.shard_rank == 0;
  const uint64_t npairs_all = membership ? 0 : (uint64_t)persons * (persons ? persons - 1 : 0) / 2 * 4 * r;
  const uint64_t npairs = rank0 ? npairs_all : 0;
  const uint64_t n = ncols * S + npairs_all;  // global lane count (all shards)
  const uint64_t W = ceil_div(n, 64);
  const uint64_t nml = shared_ml ? n : 0;
  const uint32_t nlift = V == kMpcLift ? 64u : 0u;
  const uint32_t ngates = nlift + 2u * vw.kc - 3u;
  const uint32_t ngroups = membership ? 1u : persons;
  c->query_id++;
  c->last_groups = 0;  // the AGG tap is valid only after this call's share-exact OR tree
  const uint64_t octr = ++c->or_ctr;  // fresh OR-gate streams for this query
  const uint32_t rank = c->cfg.shard_rank;
  const uint64_t s_loc = c->s;
  const uint64_t row_off = c->cfg.db_row_offset;
  static const bool serial = [] {
    const char* e = std::getenv("IRISMPC_SERIAL");  // profiling hook: no GEMM/threshold overlap
    return e && e[0] == '1';
  }();
  cudaStream_t st = c->st, st2 = (serial || c->serial) ? c->st : c->st2;
  // A/B hook IRISMPC_THR_TWO_STREAMS=1: the threshold chain's back half (lift, inject, msb) on a
  // third stream, overlapping the next job's front half (keystream, reshare) with two work-buffer
  // sets.  Measured: configs[2] 439-440 vs 425-427 ms per query on one stream, configs[1] 21.20 vs
  // 21.33 ms, so one stream is the default.
  static const bool two_thr = [] {
    const char* e = std::getenv("IRISMPC_THR_TWO_STREAMS");
    return e && e[0] == '1';
  }();
  cudaStream_t st3 = (two_thr && !serial && !c->serial) ? c->st3 : st2;
  uint64_t launches = 0;
  for (auto& e : Q.ev)
    if (!e) CK(c, cudaEventCreate(&e));
  if (!Q.done) CK(c, cudaEventCreateWithFlags(&Q.done, cudaEventDisableTiming));
  for (auto& e : c->half_free)
    if (!e) CK(c, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  for (int k = 0; k < 2; ++k) {
    if (!c->front_done[k]) CK(c, cudaEventCreateWithFlags(&c->front_done[k], cudaEventDisableTiming));
    if (!c->back_done[k]) CK(c, cudaEventCreateWithFlags(&c->back_done[k], cudaEventDisableTiming));
  }

  CK(c, cudaEventRecord(Q.ev[0], st));
  const uint8_t* dqp[3] = {dq[0], dq[1], dq[2]};
  if (host_input) {
    for (int p = 0; p < 3; ++p) {
      if (c->q_pay[p].ensure(qlen[p])) return fail(c, IRISMPC_GPU_ERR_DEVICE, "oom (query payload)");
      CK(c, cudaMemcpyAsync(c->q_pay[p].p, hq[p], qlen[p], cudaMemcpyHostToDevice, st));
      dqp[p] = c->q_pay[p].as<uint8_t>();
    }
  }
  int rc = ensure_query_buffers(c, ncols_pad);
  if (rc) return rc;
  for (auto& f : c->fld) {
    launch_parse_query_field(dqp[0], dqp[1], dqp[2], ncodes, c->l, c->l_pad, r, ncols_pad, c->shamir, f.fmt,
                             f.q.as<uint8_t>(), st);
    ++launches;
  }
  debug_check("k_parse_query_field", st);
  CK(c, cudaGetLastError());
  // rotation-pair GEMM planes (rotated queries, fields with resident S planes)
  const uint32_t npr = (r + 1) / 2;
  const uint64_t ncols_rp = (uint64_t)ncodes * npr;
  const uint32_t ncols_rp_pad = (uint32_t)round_up(ncols_rp ? ncols_rp : 1, kGemmBN);
  bool use_rp[2] = {false, false};
  for (int fi = 0; fi < 2; ++fi) {
    FieldPlanes& f = c->fld[fi];
    // the rotation-pair GEMMs run 3 products of K = l/2 over ncols_rp columns instead of one
    // of K = l over ncols: worth it only when the padded column tiles say so (batch 8:
    // 128 pair columns fill half of one 256-column tile, 1.5x the plain GEMM's tile work)
    const uint64_t bn = f.bn();
    const char* force = std::getenv("IRISMPC_RP_FORCE");  // test hook, read per query
    const bool rp_pays = 3 * ceil_div(ncols_rp, bn) < 2 * ceil_div(ncols, bn) || (force && force[0] == '1');
    use_rp[fi] = !membership && r >= 3 && (f.rpg || f.rpc) && s_loc > 0 && rp_pays;
    if (!use_rp[fi]) continue;
    const uint64_t rows = 9ull * f.nseg * f.fmt.limbs * ncols_rp_pad;  // 3 kinds x 3 parties
    const size_t bytes = rows * (c->l / 2);
    if (bytes > f.rpq.cap || f.rp_ncols_cur != ncols_rp_pad) {
      if (f.rpq.ensure(bytes)) return fail(c, IRISMPC_GPU_ERR_DEVICE, "out of device memory for RP query planes");
      CK(c, cudaMemsetAsync(f.rpq.p, 0, bytes, st));
      if (make_plane_tmap(&f.tRP, f.rpq.p, rows, c->l / 2, f.bn() / 2))
        return fail(c, IRISMPC_GPU_ERR_DEVICE, "cuTensorMapEncodeTiled failed for the RP query planes");
      f.rp_ncols_cur = ncols_rp_pad;
    }
    launch_parse_query_rp(dqp[0], dqp[1], dqp[2], ncodes, c->l, r, ncols_rp_pad, c->shamir, f.fmt,
                          f.rpq.as<uint8_t>(), st);
    ++launches;
  }
  debug_check("k_parse_query_rp", st);
  CK(c, cudaGetLastError());
  // pair dots as one limb GEMM per field: A = the unrotated query codes in the DB
  // plane layout, B = the rotated query planes (see pairs.cu).  Queued on st after
  // the DB chunks' GEMMs: the threshold chain needs them only at its end, and
  // chunk 0's GEMM starts earlier.
  auto pair_gemm = [&]() -> int {
    const uint64_t spq = round_up(ncodes, 2 * kGemmBM);
    if (Q.pair_dots.ensure(npairs * (3 * hb + fm.nparty * mb) + 64))
      return fail(c, IRISMPC_GPU_ERR_DEVICE, "oom (pair dots)");
    uint8_t* pd_out[2] = {Q.pair_dots.as<uint8_t>(), Q.pair_dots.as<uint8_t>() + 3 * npairs * hb};
    void* ph = prof_begin(st);
    for (int fi = 0; fi < 2; ++fi) {
      FieldPlanes& f = c->fld[fi];
      const uint64_t rows = (uint64_t)f.nparty * f.fmt.limbs * spq;
      if (spq != f.qa_spad) {
        if (f.qa.ensure(rows * c->l_pad)) return fail(c, IRISMPC_GPU_ERR_DEVICE, "oom (pair planes)");
        CK(c, cudaMemsetAsync(f.qa.p, 0, rows * c->l_pad, st));
        if (make_plane_tmap(&f.tQA, f.qa.p, rows, c->l_pad, kGemmBM))
          return fail(c, IRISMPC_GPU_ERR_DEVICE, "cuTensorMapEncodeTiled failed for the pair planes");
        f.qa_spad = spq;
      }
      for (uint32_t p = 0; p < f.nparty; ++p)
        launch_parse_field(dqp[p], ncodes, 0, c->l, c->l_pad, spq, (int)p, c->shamir, f.fmt, f.qa.as<uint8_t>(), st);
      if (f.pair_c.ensure(f.nparty * ncols * ncodes * f.out_bytes + 16))
        return fail(c, IRISMPC_GPU_ERR_DEVICE, "oom (pair dots)");
      GemmArgs pg = field_gemm_args(c, f, ncols_pad);
      pg.s_pad = (uint32_t)spq;
      pg.s_valid = ncodes;
      pg.ncols = (uint32_t)ncols;
      pg.out = f.pair_c.p;
      pg.out_pstride = ncols * ncodes;
      pg.out_cstride = ncodes;
      launch_gemm(f.tQA, f.tB, pg, (uint32_t)(spq / kGemmBM), (uint32_t)ceil_div(ncols, f.bn()), st);
      launch_pair_gather(f.pair_c.p, f.out_bytes, f.nparty, ncodes, (uint32_t)ncols, persons, r, pd_out[fi], npairs,
                         st);
      launches += f.nparty + 2;  // parse + gemm + gather
    }
    prof_end(ph, "pairs (gemm+gather)", st);
    debug_check("pairs", st);
    CK(c, cudaGetLastError());
    return 0;
  };
  CK(c, cudaEventRecord(Q.ev[1], st));

  const bool row_taps = c->tap_k > 0;
  if (row_taps) {  // compact L1 taps: [p][col * k + i] then the pair lanes
    const uint64_t nt = ncols * c->tap_k + npairs;
    c->tap_n = nt;
    const size_t tb[2] = {3 * nt * hb, fm.nparty * nt * mb};
    for (int t = 0; t < 7; ++t) {
      c->tap_bytes[t] = t < 2 ? tb[t] : 0;
      if (t >= 2) continue;
      if (c->tap_buf[t].ensure(tb[t] + 16)) return fail(c, IRISMPC_GPU_ERR_DEVICE, "oom (row taps)");
      CK(c, cudaMemsetAsync(c->tap_buf[t].p, 0, tb[t] + 16, st));
    }
  } else if (c->taps) {
    c->tap_n = n;
    const size_t tb[7] = {3 * n * hb, fm.nparty * n * mb, 3 * n * 4, 3 * n * 4, 3 * n * 4, 3 * n * 4, 3 * n};
    for (int t = 0; t < 7; ++t) {
      c->tap_bytes[t] = tb[t];
      if (c->tap_buf[t].ensure(tb[t] + 16)) return fail(c, IRISMPC_GPU_ERR_DEVICE, "oom (taps)");
      CK(c, cudaMemsetAsync(c->tap_buf[t].p, 0, tb[t] + 16, st));
    }
  }

  // ---- row-chunk plan
  uint64_t rows_chunk = 0, nchunks = 0;
  if (s_loc && ncols) {
    static const uint64_t target_env = [] {
      const char* e = std::getenv("IRISMPC_CHUNK_LANES");  // test hook
      return e ? std::strtoull(e, nullptr, 10) : 0ull;
    }();
    // 2^24 lanes per chunk; with the rotation-pair GEMMs, whose chunks are 25% shorter, 2^25 and at
    // least 16384 rows (wide batches: longer segments, fewer partial 1024-lane threshold tasks;
    // -1..-2% at configs[1], -5% at 128 / 256 codes)
    // Plain GEMM: 2^24 lanes, up to 2^26 on large DBs (at least 16 chunks; 1M rows x 64 codes:
    // 458 -> 430 ms per query, the per-chunk threshold ramp-up paid 4x less often; x 32 codes -1.3%,
    // x 8 codes +4% with 2^26, so small batches keep 2^24)
    const bool rp_any = use_rp[0] || use_rp[1];
    const uint64_t lanes_all = s_loc * ncols;
    const uint64_t target =
        target_env ? target_env
        : rp_any   ? std::max<uint64_t>(1ull << 25, 16384ull * ncols)
                   : std::min<uint64_t>(1ull << 26, std::max<uint64_t>(1ull << 24, lanes_all / 16));
    // Row granule: a chunk's (problem, 256-row block) units should fill whole
    // waves of the persistent GEMM's cluster groups, for every field.
    uint64_t granule = 2 * kGemmBM;
    static const bool no_granule = std::getenv("IRISMPC_NO_GRANULE") != nullptr;  // A/B hook
    for (int fi = 0; fi < 2; ++fi) {
      const FieldPlanes& f = c->fld[fi];
      if (no_granule) break;
      const uint64_t g = gemm_groups((uint32_t)ceil_div(use_rp[fi] ? ncols_rp : ncols, f.bn()));
      uint64_t a = g, b = f.nparty * (use_rp[fi] ? 3 : 1);  // m_pairs multiple of g / gcd(g, nprob)
      while (b) {
        const uint64_t t = a % b;
        a = b;
        b = t;
      }
      const uint64_t need = 2 * kGemmBM * (g / a);
      uint64_t x = granule, y = need;  // lcm(granule, need)
      while (y) {
        const uint64_t t = x % y;
        x = y;
        y = t;
      }
      granule = granule / x * need;
    }
    rows_chunk = round_up(std::max<uint64_t>(target / ncols, 1), granule);
    nchunks = ceil_div(s_loc, rows_chunk);
    // equal chunks (the last one takes the remainder)
    rows_chunk = std::min<uint64_t>(round_up(ceil_div(s_loc, nchunks), granule), round_up(s_loc, 2 * kGemmBM));
    nchunks = ceil_div(s_loc, rows_chunk);
  }
  // Chunk 0's GEMM runs alone (the threshold has nothing to do yet), so chunk 0
  // is cut to a quarter and the threshold chain starts early (measured -1.7%;
  // geometric ramps of the following chunk sizes were slower).
  std::vector<uint64_t> chunk_row0;
  if (nchunks) {
    static const double head_div = [] {  // A/B hooks: head fraction and growth ratio
      const char* e = std::getenv("IRISMPC_HEAD_DIV");
      return e ? std::atof(e) : 4.0;
    }();
    static const double ramp = [] {
      const char* e = std::getenv("IRISMPC_RAMP");
      return e ? std::atof(e) : 100.0;
    }();
    uint64_t len = rows_chunk;
    if (nchunks >= 2 && head_div > 1.0)
      len = std::max<uint64_t>(2 * kGemmBM, round_up((uint64_t)(rows_chunk / head_div), 2 * kGemmBM));
    for (uint64_t r0 = 0; r0 < s_loc;) {
      chunk_row0.push_back(r0);
      r0 += len;
      len = std::min<uint64_t>(rows_chunk, round_up((uint64_t)(len * ramp), 2 * kGemmBM));
    }
    nchunks = chunk_row0.size();
    chunk_row0.push_back(s_loc);
  }
  auto chunk_rows = [&](uint64_t i) { return std::min<uint64_t>(chunk_row0[i + 1], s_loc) - chunk_row0[i]; };
  auto seg_tasks = [](uint64_t lb, uint64_t le) { return (le - 1) / 1024 - lb / 1024 + 1; };
  // fused-OR slots of the bucketed OR (DB-sharded queries; the share-exact tree of
  // unsharded queries reads the match words instead): per column contiguous (all its
  // lanes belong to one person)
  std::vector<uint64_t> col_slot(ncols + 1, 0);
  uint64_t total_slots = 0;
  for (uint64_t col = 0; col < ncols; ++col) {
    col_slot[col] = total_slots;
    for (uint64_t i = 0; i < nchunks; ++i) {
      const uint64_t lb = col * S + row_off + chunk_row0[i];
      total_slots += seg_tasks(lb, lb + chunk_rows(i));
    }
  }
  col_slot[ncols] = total_slots;
  std::vector<uint64_t> h_slot_begin(ngroups + 1);
  for (uint32_t g = 0; g <= ngroups; ++g)
    h_slot_begin[g] = membership ? (g == 0 ? 0 : total_slots) : col_slot[(uint64_t)g * 2 * r];
  {
    const uint64_t per_person_max = total_slots + npairs_all;  // linear OR items of one person, at most
    if (per_person_max >= kOrTreeOffset || ngroups >= (1u << 23))
      return fail(c, IRISMPC_GPU_ERR_BOUNDS, "OR-gate stream windows exceeded (persons >= 2^23 or 2^39 items)");
  }
  if (c->partial.ensure(3 * total_slots + 16) || Q.slot_begin.ensure((ngroups + 1) * sizeof(uint64_t)) ||
      c->person_out.ensure(3ull * ngroups + 16))
    return fail(c, IRISMPC_GPU_ERR_DEVICE, "oom (or buffers)");
  CK(c, cudaMemcpyAsync(Q.slot_begin.p, h_slot_begin.data(), (ngroups + 1) * sizeof(uint64_t),
                        cudaMemcpyHostToDevice, st));

  const bool dbg = c->cfg.debug_rows != 0 && row_bits_out;
  // the reference's own OR tree over every lane's bit (share-exact) for an unsharded
  // query; DB-sharded queries keep the bucketed per-shard OR (the reference has no shards)
  static const bool or_bucketed = [] {  // A/B hook
    const char* e = std::getenv("IRISMPC_OR_TREE");
    return e && std::string(e) == "bucketed";
  }();
  const bool exact_or = mode == 0 && S == s_loc && row_off == 0 && !or_bucketed;
  uint64_t match_w0 = 0, match_words = 0;
  if (dbg || exact_or) {
    match_words = 2 * ceil_div(n, 64) + 4;  // + padding for the tree's 64-bit funnel reads
  } else if (npairs) {
    match_w0 = (ncols * S) / 32;
    match_words = ceil_div(n, 32) - match_w0 + 1;
  }
  for (int p = 0; p < 3 && match_words; ++p) {
    if (Q.match[p].ensure(match_words * 4)) return fail(c, IRISMPC_GPU_ERR_DEVICE, "oom (match)");
    CK(c, cudaMemsetAsync(Q.match[p].p, 0, match_words * 4, st));
  }

  // ---- segments [chunk][col] then the pair segment; jobs group segments
  struct Job {
    uint64_t seg0, nseg, ntasks, ngrp, ngblk, gwords, chunk, ks_seg, grp_seg, task_seg;
    bool pair;
  };
  std::vector<Job> jobs;
  const uint64_t nsegs_all = nchunks * ncols + (npairs ? 1 : 0);
  if (nsegs_all + 1 > Q.h_segs_cap) {
    if (Q.h_segs) cudaFreeHost(Q.h_segs);
    Q.h_segs = nullptr;
    Q.h_segs_cap = 0;
    CK(c, cudaMallocHost(&Q.h_segs, (nsegs_all + 1) * sizeof(Seg)));
    Q.h_segs_cap = nsegs_all + 1;
  }
  Seg* const hsegs = Q.h_segs;
  if (Q.segs.ensure((nsegs_all + 1) * sizeof(Seg))) return fail(c, IRISMPC_GPU_ERR_DEVICE, "oom (segs)");
  auto add_job = [&](uint64_t seg0, uint64_t nseg, bool pair, uint64_t chunk) {
    Job j{seg0, nseg, 0, 0, 0, 0, chunk, 0, 0, 0, pair};
    for (uint64_t i = seg0; i < seg0 + nseg; ++i) {
      Seg& sg = hsegs[i];
      sg.q_first = sg.lane_begin / 1024;
      sg.w_first = sg.lane_begin / 64;
      sg.task_begin = j.ntasks;
      sg.grp_begin = j.ngrp;
      sg.gblk_begin = j.ngblk;
      sg.g_off = j.gwords;
      const uint64_t nw = (sg.lane_end - 1) / 64 - sg.w_first + 1;
      j.ntasks += seg_tasks(sg.lane_begin, sg.lane_end);
      j.ngrp += (sg.lane_end - 1) / 8 - sg.lane_begin / 8 + 1;
      j.task_seg = std::max<uint64_t>(j.task_seg, seg_tasks(sg.lane_begin, sg.lane_end));
      j.grp_seg = std::max<uint64_t>(j.grp_seg, (sg.lane_end - 1) / 8 - sg.lane_begin / 8 + 1);
      j.ngblk += 3ull * ngates * (nw / 8 + 2);
      j.ks_seg = std::max<uint64_t>(j.ks_seg, 3ull * ngates * (nw / 8 + 2));
      j.gwords += 3ull * ngates * gate_row_words(nw);
    }
    jobs.push_back(j);
  };
  static const uint64_t kThrLanes = [] {
    const char* e = std::getenv("IRISMPC_THR_LANES");  // test hook: force multi-job splits
    return e ? std::strtoull(e, nullptr, 10) : (1ull << 26);
  }();
  uint64_t cstride = 0;
  {
    std::vector<uint64_t> col_fill(col_slot.begin(), col_slot.end());
    for (uint64_t i = 0; i < nchunks; ++i) {
      const uint64_t nr = chunk_rows(i);
      for (uint64_t col = 0; col < ncols; ++col) {
        Seg& sg = hsegs[i * ncols + col];
        sg.lane_begin = col * S + row_off + chunk_row0[i];
        sg.lane_end = sg.lane_begin + nr;
        sg.src = col * nr;
        sg.src_rp = ((col / r) * npr + (col % r) / 2) * nr;  // RP: the rotation pair's P planes
        sg.rp_sel = ((col % r) & 1) ? 1u : 2u;
        sg.slot = exact_or ? -1 : (int64_t)col_fill[col];
        col_fill[col] += seg_tasks(sg.lane_begin, sg.lane_end);
      }
      // threshold jobs of at most kThrLanes lanes (plus 1/8 slack: a chunk rounded up to its row
      // granule stays one job), the columns split evenly (no small remainder job)
      const uint64_t njobs_c = ceil_div(ncols * nr, kThrLanes + kThrLanes / 8);
      const uint64_t per_job = std::max<uint64_t>(1, ceil_div(ncols, std::max<uint64_t>(1, njobs_c)));
      for (uint64_t a = 0; a < ncols; a += per_job)
        add_job(i * ncols + a, std::min<uint64_t>(per_job, ncols - a), false, i);
      cstride = std::max<uint64_t>(cstride, ncols * nr);
    }
  }
  if (npairs) {
    Seg& sg = hsegs[nsegs_all - 1];
    sg.lane_begin = ncols * S;
    sg.lane_end = n;
    sg.src = 0;
    sg.src_rp = 0;
    sg.rp_sel = 0;
    sg.slot = -1;
    add_job(nsegs_all - 1, 1, true, 0);
    cstride = std::max<uint64_t>(cstride, npairs);
  }
  cstride = round_up(cstride, 8);  // 16-byte aligned component planes
  uint64_t max_g = 0, max_bits = 0;
  for (const Job& j : jobs) {
    max_g = std::max(max_g, j.gwords);
    max_bits = std::max(max_bits, j.ntasks * 32);
  }
  // dot buffers the GEMM stream rotates through (2: the GEMM runs at most one chunk ahead of
  // the threshold; IRISMPC_DOT_BUFS=3|4: A/B hook)
  static const int ndotbufs = [] {
    const char* e = std::getenv("IRISMPC_DOT_BUFS");
    return e ? std::max(2, std::min(irismpc_gpu_ctx::kMaxDotBufs, std::atoi(e))) : 2;
  }();
  // one dot buffer: hd [3][ncols * rows_chunk] then ml [nparty][ncols * rows_chunk]
  // per field: plain [party][col][row] dots, or RP [kind P1 | P2 | P3][party][rotation pair][row]
  const uint64_t hcols = use_rp[0] ? 3 * ncols_rp : ncols, mcols = use_rp[1] ? 3 * ncols_rp : ncols;
  const uint64_t hd_half = 3 * hcols * rows_chunk * hb;
  const uint64_t dots_half = round_up(hd_half + fm.nparty * mcols * rows_chunk * mb, 16);
  if (nsegs_all) {
    CK(c, cudaMemcpyAsync(Q.segs.p, hsegs, nsegs_all * sizeof(Seg), cudaMemcpyHostToDevice, st));
    if (nchunks && c->dots.ensure(ndotbufs * dots_half)) return fail(c, IRISMPC_GPU_ERR_DEVICE, "oom (dot buffers)");
    for (int k = 0; k < (st3 != st2 ? 2 : 1); ++k)
      if (c->wk_ml_rs[k].ensure((V == kMpcLift ? 3 * cstride * sizeof(uint16_t) : 0) + 16) ||
          c->wk_diff[k].ensure(3 * cstride * sizeof(uint32_t) + 16) ||
          c->wk_gate[k].ensure(max_g * sizeof(uint64_t) + 16) ||
          c->wk_bits[k].ensure((V == kMpcLift ? 6 * max_bits * sizeof(uint32_t) : 0) + 16))
        return fail(c, IRISMPC_GPU_ERR_DEVICE, "oom (threshold work buffers)");
  }
  // per-chunk S planes (IRISMPC_RP_CHUNKED): one scratch per field, reused chunk after chunk on
  // the GEMM stream (k_rp_sum of chunk i+1 is queued behind chunk i's GEMM)
  for (int fi = 0; fi < 2; ++fi) {
    FieldPlanes& f = c->fld[fi];
    if (!use_rp[fi] || f.rpg || f.rpconv) continue;
    uint64_t spad = 0;
    for (uint64_t i = 0; i < nchunks; ++i) spad = std::max<uint64_t>(spad, round_up(chunk_rows(i), 2 * kGemmBM));
    if (spad > f.sch_spad) {
      const uint64_t rows = (uint64_t)f.nparty * f.fmt.limbs * spad;
      if (f.sch.ensure(rows * (c->l / 2))) return fail(c, IRISMPC_GPU_ERR_DEVICE, "oom (per-chunk RP sum planes)");
      if (make_plane_tmap(&f.tSc, f.sch.p, rows, c->l / 2, kGemmBM))
        return fail(c, IRISMPC_GPU_ERR_DEVICE, "cuTensorMapEncodeTiled failed for the per-chunk RP sum planes");
      f.sch_spad = spad;
    }
  }

  ThrArgs ta{};
  ta.variant = V;
  ta.n = n;
  ta.W = W;
  ta.tile_kernels = c->thr_tile;
  for (int k = 0; k < 3; ++k) {
    ta.pos[k] = c->pos[k];
    ta.key[k] = c->keys[k];
    // stream layout: reshare n (+ n), lift 64W + inject, msb
    const uint64_t inj = V == kMpcLift ? 64 * W + (k == 0 ? 2 * n : (k == 1 ? 0 : 6 * n)) : 0;
    ta.lift_base[k] = c->pos[k] + n + nml;
    ta.inj_base[k] = ta.lift_base[k] + 64 * W;
    ta.msb_base[k] = c->pos[k] + n + nml + inj;
  }
  ta.nlift = nlift;
  ta.ngates = ngates;
  ta.a = c->cfg.a;
  ta.b = c->cfg.b;
  ta.coef = 1.0 - 2.0 * c->cfg.match_ratio;
  ta.partial = c->partial.as<uint8_t>();
  ta.nslots = total_slots;
  ta.or_stream = or_stream_id(octr, rank, 1);
  ta.or_elem_base = 0;
  ta.cstride = cstride;
  if (c->taps && !row_taps) {
    ta.tap_rs_hd = c->tap_buf[2].as<uint32_t>();
    ta.tap_rs_ml = c->tap_buf[3].as<uint32_t>();
    ta.tap_ml32 = c->tap_buf[4].as<uint32_t>();
    ta.tap_diff = c->tap_buf[5].as<uint32_t>();
    ta.tap_msb = c->tap_buf[6].as<uint8_t>();
  }
  uint64_t task_off = 0;
  // hd_base: [3][pstride] hd dots; ml_base: [nparty][pstride] ml dots / public popcounts
  auto run_job = [&](const Job& j, const uint8_t* hd_base, const uint8_t* ml_base, uint64_t pstride_h,
                     uint64_t pstride_m, uint64_t ks_h, uint64_t ks_m) -> int {
    ThrArgs t = ta;
    t.segs = Q.segs.as<Seg>() + j.seg0;
    t.nsegs = (uint32_t)j.nseg;
    t.ntasks = j.ntasks;
    t.ngrp = j.ngrp;
    t.ngblk = j.ngblk;
    t.ks_seg_threads = (uint32_t)j.ks_seg;
    t.grp_seg_max = (uint32_t)j.grp_seg;
    t.task_seg_max = (uint32_t)j.task_seg;
    // work-buffer set of this job: front (st2) waits until the back half (st3) of the job
    // two before, which used the same set, is done; back waits for this job's front
    const int wp = st3 != st2 ? (int)(c->job_ctr++ % 2) : 0;
    t.ml_rs = c->wk_ml_rs[wp].as<uint16_t>();
    t.diff = c->wk_diff[wp].as<uint32_t>();
    t.gate = c->wk_gate[wp].as<uint64_t>();
    t.bits = c->wk_bits[wp].as<uint32_t>();
    t.nbits = j.ntasks * 32;
    t.or_elem_base = ta.or_elem_base + task_off * 64;
    task_off += j.ntasks;
    for (int p = 0; p < 3; ++p) {
      t.hd[p] = hd_base + p * pstride_h * hb;
      t.ml[p] = ml_base + (fm.nparty == 3 ? p : 0) * pstride_m * mb;
      t.match[p] = (j.pair || dbg || exact_or) ? Q.match[p].as<uint32_t>() : nullptr;
    }
    t.match_w0 = j.pair ? match_w0 : 0;
    t.rp_kstride_h = ks_h;
    t.rp_kstride_m = ks_m;
    if (st3 != st2) CK(c, cudaStreamWaitEvent(st2, c->back_done[wp], 0));
    launch_threshold_front(t, st2);
    if (st3 != st2) {
      CK(c, cudaEventRecord(c->front_done[wp], st2));
      CK(c, cudaStreamWaitEvent(st3, c->front_done[wp], 0));
    }
    launch_threshold_back(t, st3);
    if (st3 != st2) CK(c, cudaEventRecord(c->back_done[wp], st3));
    CK(c, cudaGetLastError());
    launches += V == kMpcLift ? 5 : 3;
    return 0;
  };
  auto ensure_events = [&](std::vector<cudaEvent_t>& v, size_t n_) -> int {
    while (v.size() < n_) {
      cudaEvent_t e;
      CK(c, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      v.push_back(e);
    }
    return 0;
  };
  if (ensure_events(c->evg, nchunks + 1) || ensure_events(c->evt, 1)) return IRISMPC_GPU_ERR_DEVICE;
  while (Q.gev.size() < 2 * nchunks) {
    cudaEvent_t e;
    CK(c, cudaEventCreate(&e));
    Q.gev.push_back(e);
  }

  // st2 starts once the prep on st (payload parse, pairs, memsets, uploads) is queued before it
  CK(c, cudaEventRecord(c->evg[nchunks], st));
  CK(c, cudaStreamWaitEvent(st2, c->evg[nchunks], 0));
  CK(c, cudaEventRecord(Q.ev[2], st2));

  // ---- DB lanes: GEMMs(i) on st || threshold(i-1) on st2
  uint64_t gemm_launches = 0;
  uint64_t gemm_ops = 0;  // executed int8 ops of the DB-lane GEMMs
  for (int fi = 0; fi < 2; ++fi) {
    const FieldPlanes& f = c->fld[fi];
    const uint64_t L = (uint64_t)f.fmt.limbs, prods = L * (L + 1) / 2;
    gemm_ops += use_rp[fi] ? 2 * prods * 3 * f.nparty * ncols_rp * s_loc * (c->l / 2) * f.nseg
                           : 2 * prods * f.nparty * ncols * s_loc * c->l_pad * f.nseg;
  }
  size_t ji = 0;
  for (uint64_t i = 0; i < nchunks; ++i) {
    const uint64_t nr = chunk_rows(i);
    // dot-buffer halves alternate across chunks and across queries: the GEMM
    // waits for the threshold of the last chunk (of any query) that read the half
    const int half = (int)(c->chunk_ctr++ % ndotbufs);
    uint8_t* dots = c->dots.as<uint8_t>() + half * dots_half;
    uint8_t* dots_ml = dots + hd_half;
    CK(c, cudaStreamWaitEvent(st, c->half_free[half], 0));
    CK(c, cudaEventRecord(Q.gev[2 * i], st));
    for (int fi = 0; fi < 2; ++fi) {
      FieldPlanes& f = c->fld[fi];
      const uint32_t m_tiles = (uint32_t)(round_up(nr, 2 * kGemmBM) / kGemmBM);
      void* ph = prof_begin(st);
      if (use_rp[fi]) {
        // P1 = E.D0, P2 = S.M, P3 = O.D1 over half-length K (prep.cu, rotation pairs)
        // one launch, 3 kinds x 3 parties: fewer partial last waves than three launches
        GemmArgs g = field_gemm_args(c, f, ncols_rp_pad);
        g.nkb_seg = (c->l / 2) / kGemmBK;
        g.nkind = 3;
        g.a_kb0_k2 = (c->l / 2) / kGemmBK;
        g.b_kind_rows = (uint32_t)(3ull * f.nseg * f.fmt.limbs * ncols_rp_pad);
        g.s_pad = (uint32_t)c->s_pad;
        g.s_valid = (uint32_t)nr;
        g.row0 = (uint32_t)chunk_row0[i];
        g.ncols = (uint32_t)ncols_rp;
        g.out = fi == 0 ? dots : dots_ml;
        g.out_pstride = ncols_rp * nr;
        g.out_kstride = 3 * ncols_rp * nr;
        g.out_cstride = (uint32_t)nr;
        if (!f.rpg && f.rpconv) {
          g.s_conv = 1;  // S = E + O in the GEMM's shared memory
        } else if (!f.rpg) {  // per-chunk S planes: E + O of this chunk's rows, then the GEMM (same stream)
          const uint64_t nrs = std::min<uint64_t>(round_up(nr, 2 * kGemmBM), c->s_pad - chunk_row0[i]);
          launch_rp_sum_rows(f.db.as<uint8_t>(), f.nparty, c->s_pad, chunk_row0[i], nrs, f.sch_spad, c->l,
                             c->l_pad, f.fmt.limbs, f.sch.as<uint8_t>(), st);
          ++launches;
          g.s_pad2 = (uint32_t)f.sch_spad;
          g.row0_2 = 0;
        }
        launch_gemm(f.tA, f.tRP, g, m_tiles, (uint32_t)ceil_div(ncols_rp, f.bn()), st,
                    f.rpg ? &f.tS : (f.rpconv ? &f.tA : &f.tSc));
        ++gemm_launches;
        ++launches;
      } else {
        GemmArgs g = field_gemm_args(c, f, ncols_pad);
        g.s_pad = (uint32_t)c->s_pad;
        g.s_valid = (uint32_t)nr;
        g.row0 = (uint32_t)chunk_row0[i];
        g.ncols = (uint32_t)ncols;
        g.out = fi == 0 ? dots : dots_ml;
        g.out_pstride = ncols * nr;
        g.out_cstride = (uint32_t)nr;
        launch_gemm(f.tA, f.tB, g, m_tiles, (uint32_t)ceil_div(ncols, f.bn()), st);
        ++gemm_launches;
        ++launches;
      }
      prof_end(ph, fi == 0 ? "k_limb_gemm_pair (hd)" : "k_limb_gemm_pair (ml)", st);
      debug_check("k_limb_gemm_pair", st);
      CK(c, cudaGetLastError());
    }
    CK(c, cudaEventRecord(Q.gev[2 * i + 1], st));
    if (row_taps) {
      const uint64_t nt = c->tap_n;
      launch_tap_rows(dots, (int)hb, 3, ncols, r, nr, use_rp[0] ? 3 * ncols_rp * nr : 0,
                      c->tap_rows_dev.as<uint64_t>(), c->tap_k, chunk_row0[i], c->tap_buf[0].p, nt, st);
      launch_tap_rows(dots_ml, (int)mb, fm.nparty, ncols, r, nr, use_rp[1] ? 3 * ncols_rp * nr : 0,
                      c->tap_rows_dev.as<uint64_t>(), c->tap_k, chunk_row0[i], c->tap_buf[1].p, nt, st);
      CK(c, cudaGetLastError());
    } else if (c->taps && c->cfg.db_rows_total == 0) {
      // L1 tap: dots[(col, row - r0)] -> lane col*S + row
      if (use_rp[0])
        launch_rp_tap(dots, (int)hb, 3, ncols, r, nr, 3 * ncols_rp * nr, c->tap_buf[0].p, n, S, chunk_row0[i], st);
      else
        for (uint32_t p = 0; p < 3; ++p)
          CK(c, cudaMemcpy2DAsync(c->tap_buf[0].as<uint8_t>() + (p * n + chunk_row0[i]) * hb, S * hb,
                                  dots + p * ncols * nr * hb, nr * hb, nr * hb, ncols, cudaMemcpyDeviceToDevice, st));
      if (use_rp[1])
        launch_rp_tap(dots_ml, (int)mb, 3, ncols, r, nr, 3 * ncols_rp * nr, c->tap_buf[1].p, n, S, chunk_row0[i],
                      st);
      else
        for (uint32_t p = 0; p < fm.nparty; ++p)
          CK(c, cudaMemcpy2DAsync(c->tap_buf[1].as<uint8_t>() + (p * n + chunk_row0[i]) * mb, S * mb,
                                  dots_ml + p * ncols * nr * mb, nr * mb, nr * mb, ncols, cudaMemcpyDeviceToDevice,
                                  st));
    }
    CK(c, cudaEventRecord(c->evg[i], st));
    CK(c, cudaStreamWaitEvent(st2, c->evg[i], 0));
    for (; ji < jobs.size() && !jobs[ji].pair && jobs[ji].chunk == i; ++ji) {
      const uint64_t rpn = ncols_rp * nr;
      int rc2 = run_job(jobs[ji], dots, dots_ml, use_rp[0] ? rpn : ncols * nr, use_rp[1] ? rpn : ncols * nr,
                        use_rp[0] ? 3 * rpn : 0, use_rp[1] ? 3 * rpn : 0);
      if (rc2) return rc2;
    }
    CK(c, cudaEventRecord(c->half_free[half], st2));
  }

  // ---- pair lanes (shard 0): pair GEMMs on st, then their threshold into match words on st2
  if (npairs) {
    const int prc = pair_gemm();
    if (prc) return prc;
    CK(c, cudaEventRecord(Q.ev[5], st));
    CK(c, cudaStreamWaitEvent(st2, Q.ev[5], 0));
  }
  if (npairs) {
    const uint8_t* pd_hd = Q.pair_dots.as<uint8_t>();
    const uint8_t* pd_ml = pd_hd + 3 * npairs * hb;
    if (row_taps) {
      const uint64_t nt = c->tap_n, o = ncols * c->tap_k;
      for (uint32_t p = 0; p < 3; ++p)
        CK(c, cudaMemcpyAsync(c->tap_buf[0].as<uint8_t>() + (p * nt + o) * hb, pd_hd + p * npairs * hb, npairs * hb,
                              cudaMemcpyDeviceToDevice, st2));
      for (uint32_t p = 0; p < fm.nparty; ++p)
        CK(c, cudaMemcpyAsync(c->tap_buf[1].as<uint8_t>() + (p * nt + o) * mb, pd_ml + p * npairs * mb, npairs * mb,
                              cudaMemcpyDeviceToDevice, st2));
    } else if (c->taps && c->cfg.db_rows_total == 0) {
      for (uint32_t p = 0; p < 3; ++p)
        CK(c, cudaMemcpyAsync(c->tap_buf[0].as<uint8_t>() + (p * n + ncols * S) * hb, pd_hd + p * npairs * hb,
                              npairs * hb, cudaMemcpyDeviceToDevice, st2));
      for (uint32_t p = 0; p < fm.nparty; ++p)
        CK(c, cudaMemcpyAsync(c->tap_buf[1].as<uint8_t>() + (p * n + ncols * S) * mb, pd_ml + p * npairs * mb,
                              npairs * mb, cudaMemcpyDeviceToDevice, st2));
    }
    int rc2 = run_job(jobs.back(), pd_hd, pd_ml, npairs, npairs, 0, 0);
    if (rc2) return rc2;
  }
  if (st3 != st2) {  // the OR reads every job's partial slots (written by the back halves)
    CK(c, cudaEventRecord(c->evt[0], st3));
    CK(c, cudaStreamWaitEvent(st2, c->evt[0], 0));
  }
  CK(c, cudaEventRecord(Q.ev[3], st2));

  // ---- per-person OR (st2), then the open on st
  if (exact_or) {
    OrTreeArgs oa{};
    for (int p = 0; p < 3; ++p) oa.match[p] = Q.match[p].as<uint64_t>();
    oa.ngroups = ngroups;
    oa.db_lanes = membership ? S : 2ull * r * S;
    oa.pair_base = ncols * S;
    oa.pair_block = npairs ? 4ull * r : 0;
    oa.lanes = oa.db_lanes + (npairs ? (uint64_t)(ngroups - 1) * 4 * r : 0);
    for (int k = 0; k < 3; ++k) oa.key[k] = c->keys[k];
    uint64_t rs[3];
    for (int k = 0; k < 3; ++k) rs[k] = ta.msb_base[k] + (uint64_t)(2 * vw.kc - 3) * W;
    const uint64_t words = ortree_scratch_words(ngroups, oa.lanes);
    if (c->or_scr[0].ensure(words * 8) || c->or_scr[1].ensure(words * 8))
      return fail(c, IRISMPC_GPU_ERR_DEVICE, "oom (or tree)");
    uint64_t* scr[2] = {c->or_scr[0].as<uint64_t>(), c->or_scr[1].as<uint64_t>()};
    void* ph2 = prof_begin(st2);
    launches += launch_ortree(oa, rs, scr, c->person_out.as<uint8_t>(), st2);
    c->last_groups = ngroups;
    prof_end(ph2, "k_ortree", st2);
    debug_check("k_ortree", st2);
    CK(c, cudaGetLastError());
  } else {
  OrArgs oa{};
  oa.partial = c->partial.as<uint8_t>();
  oa.nslots = total_slots;
  oa.slot_begin = Q.slot_begin.as<uint64_t>();
  for (int p = 0; p < 3; ++p) oa.pair_match[p] = npairs ? Q.match[p].as<uint32_t>() : nullptr;
  oa.pair_w0 = match_w0;
  oa.pair_lane0 = ncols * S;
  oa.persons = ngroups;
  oa.rot = r;
  for (int k = 0; k < 3; ++k) oa.key[k] = c->keys[k];
  oa.stream = or_stream_id(octr, rank, 2);
  oa.out = c->person_out.as<uint8_t>();
  void* ph2 = prof_begin(st2);
  launch_or_persons(oa, st2);
  prof_end(ph2, "k_or_persons", st2);
  debug_check("k_or_persons", st2);
  CK(c, cudaGetLastError());
  ++launches;
  }
  // the open (mode 0) or the partial hand-off (mode 1) also on the threshold
  // stream, so the GEMM stream is free for the next query's chunks
  if (mode == 0) {
    if (Q.open_out.ensure(ngroups + 16)) return fail(c, IRISMPC_GPU_ERR_DEVICE, "oom");
    if (ngroups + 16 > Q.h_match_cap) {
      if (Q.h_match) cudaFreeHost(Q.h_match);
      Q.h_match = nullptr;
      Q.h_match_cap = 0;
      CK(c, cudaMallocHost(&Q.h_match, ngroups + 16));
      Q.h_match_cap = ngroups + 16;
    }
    launch_or_open(c->person_out.as<uint8_t>(), 1, ngroups, c->keys, or_stream_id(octr, rank, 3),
                   Q.open_out.as<uint8_t>(), st2);
    CK(c, cudaGetLastError());
    ++launches;
    CK(c, cudaMemcpyAsync(Q.h_match, Q.open_out.p, ngroups, cudaMemcpyDeviceToHost, st2));
  } else {
    CK(c, cudaMemcpyAsync(partial_dev, c->person_out.p, 3ull * ngroups, cudaMemcpyDeviceToDevice, st2));
  }
  CK(c, cudaEventRecord(Q.ev[4], st2));
  CK(c, cudaEventRecord(Q.done, st2));
  Q.inflight = true;
  Q.ticket = ++c->tickets;
  Q.mode = mode;
  Q.ngroups = ngroups;
  Q.match_out = match_out;
  Q.row_bits_out = dbg ? row_bits_out : nullptr;
  Q.n = n;
  Q.nchunks = nchunks;
  c->par ^= 1;

  // ---- advance the seed streams exactly as the reference does (A.3)
  const uint64_t glen = membership ? S : 2ull * r * S + (uint64_t)(persons ? persons - 1 : 0) * 4 * r;
  uint64_t or_rounds = 0, or_bytes = 0;
  const uint64_t ord = ref_or_draws(ngroups, glen, &or_rounds, &or_bytes);
  const uint64_t msb_draws = (uint64_t)(2 * vw.kc - 3) * W;
  for (int k = 0; k < 3; ++k) c->pos[k] = ta.msb_base[k] + msb_draws + ord;

  {
    irismpc_gpu_stats* st_ = &Q.stats;
    std::memset(st_, 0, sizeof(*st_));
    st_->s = S;
    st_->l = c->l;
    st_->batch = membership ? 1 : persons;
    st_->lanes = n;
    const uint64_t nb8 = ceil_div(n, 8), open_b = ceil_div(ngroups, 8);
    for (int p = 0; p < 3; ++p) {
      st_->dot_bytes[p] = n * (vw.kh / 8) + nml * (vw.km / 8);
      st_->lift_bytes[p] = V == kMpcLift ? 64 * nb8 + (p == 0 ? 8 * n : 4 * n) : 0;
      st_->msb_bytes[p] = (uint64_t)(2 * vw.kc - 3) * nb8;
      st_->or_tree_bytes[p] = or_bytes + (p == 0 ? 0 : open_b) + (c->cfg.debug_rows && p != 0 ? nb8 : 0);
    }
    st_->dot_rounds = 1;
    st_->lift_rounds = V == kMpcLift ? 21 : 0;
    st_->msb_rounds = (uint64_t)vw.kc - 1;
    st_->or_tree_rounds = or_rounds + 1 + (c->cfg.debug_rows ? 1 : 0);
    st_->gemm_launches = gemm_launches;
    st_->kernel_launches = launches;
    st_->gemm_int8_ops = gemm_ops;
    st_->rotation_pair_gemm = (use_rp[0] || use_rp[1]) ? 1u : 0u;
  }
  if (ticket_out) {  // asynchronous: the caller collects with irismpc_gpu_batch_query_wait
    *ticket_out = Q.ticket;
    return 0;
  }
  const int rc_f = finish_slot(c, Q);
  if (rc_f) return rc_f;
  if (stats) *stats = Q.stats;
  return 0;
}

// Completes a slot's query: waits for its last event, copies the opened bits
// (and the debug row bits) out, fills the device times.
int finish_slot(irismpc_gpu_ctx* c, QSlot& q) {
  if (!q.inflight) return 0;
  q.inflight = false;
  CK(c, cudaEventSynchronize(q.done));
  if (q.mode == 0 && q.match_out) std::memcpy(q.match_out, q.h_match, q.ngroups);
  if (q.row_bits_out) {
    std::vector<uint32_t> w[3];
    const uint64_t nw = ceil_div(q.n, 32);
    for (int p = 0; p < 3; ++p) {
      w[p].resize(nw);
      CK(c, cudaMemcpy(w[p].data(), q.match[p].p, nw * 4, cudaMemcpyDeviceToHost));
    }
    for (uint64_t i = 0; i < q.n; ++i)
      q.row_bits_out[i] = (uint8_t)(((w[0][i / 32] ^ w[1][i / 32] ^ w[2][i / 32]) >> (i % 32)) & 1u);
  }
  float ms = 0;
  cudaEventElapsedTime(&ms, q.ev[0], q.ev[4]);
  q.stats.wall_ms = ms;
  cudaEventElapsedTime(&ms, q.ev[0], q.ev[1]);
  q.stats.prep_ms = ms;
  double gemm_ms = 0;
  for (uint64_t i = 0; i < q.nchunks; ++i) {
    cudaEventElapsedTime(&ms, q.gev[2 * i], q.gev[2 * i + 1]);
    gemm_ms += ms;
  }
  q.stats.gemm_ms = gemm_ms;
  cudaEventElapsedTime(&ms, q.ev[2], q.ev[3]);
  q.stats.threshold_ms = ms;  // stream-2 span: threshold of all chunks (overlaps the GEMMs)
  cudaEventElapsedTime(&ms, q.ev[3], q.ev[4]);
  q.stats.or_ms = ms;
  return 0;
}

// every in-flight batch query of the context (before anything that reuses its buffers)
int drain(irismpc_gpu_ctx* c) {
  for (auto& q : c->qs)
    if (q.inflight) {
      const int rc = finish_slot(c, q);
      if (rc) return rc;
    }
  return 0;
}

// The comparison phase alone: party_comparison_only / run_comparison_local
// (src/engine.cpp:448-515, src/cluster.cpp:97-145) over replicated shares of
// per-lane (masked dot, ml) values, then optionally the OR over all lanes and
// the open at P1 (with_or_tree).  Same K4 kernels as a batch query without the
// reshare (the inputs are already replicated shares), so every PRF offset is
// the batch query's minus the reshare draws.  Lanes run as jobs of at most
// 2^24 lanes on one stream.  mode 1: or_tree_only (party_or_tree_only,
// engine.cpp:517-532): hd = bit-share payload, ml unused.
int run_compare(irismpc_gpu_ctx* c, int mode, const uint8_t* const hd[3], const size_t hd_len[3],
                const uint8_t* const ml[3], const size_t ml_len[3], uint64_t n, int with_or, uint8_t* opened_out,
                uint8_t* lane_bits_out, irismpc_gpu_stats* stats) {
  if (int rc = drain(c)) return rc;
  const int V = c->variant;
  const VariantWidths vw = c->vw;
  const bool or_only = mode == 1;
  const int hw = vw.kh / 8, mw = vw.km ? vw.km / 8 : 8;
  const uint64_t W = ceil_div(n, 64);
  if (or_only) {
    for (int p = 0; p < 3; ++p)
      if (hd_len[p] != W * 16) return fail(c, IRISMPC_GPU_ERR_CONFIG, "or-tree payload size mismatch");
  } else {
    for (int p = 0; p < 3; ++p) {
      if (hd_len[p] != n * 2 * hw) return fail(c, IRISMPC_GPU_ERR_CONFIG, "bench payload size mismatch");
      if (ml_len[p] != n * (vw.km ? 2 * mw : 8)) return fail(c, IRISMPC_GPU_ERR_CONFIG, "bench ml payload size mismatch");
    }
  }
  cudaStream_t st = c->st;
  uint64_t launches = 0;
  CK(c, cudaEventRecord(c->ev[0], st));
  // inputs: H2D of the three payloads, parse into components
  Buf in_h[3], in_m[3], bad;
  const uint64_t hb = hw, mb = vw.km ? mw : 2;
  if (bad.ensure(sizeof(int))) return fail(c, IRISMPC_GPU_ERR_DEVICE, "oom");
  CK(c, cudaMemsetAsync(bad.p, 0, sizeof(int), st));
  for (int p = 0; p < 3; ++p) {
    if (in_h[p].ensure(hd_len[p] + 16)) return fail(c, IRISMPC_GPU_ERR_DEVICE, "oom (bench payload)");
    CK(c, cudaMemcpyAsync(in_h[p].p, hd[p], hd_len[p], cudaMemcpyHostToDevice, st));
    if (!or_only) {
      if (in_m[p].ensure(ml_len[p] + 16)) return fail(c, IRISMPC_GPU_ERR_DEVICE, "oom (bench payload)");
      CK(c, cudaMemcpyAsync(in_m[p].p, ml[p], ml_len[p], cudaMemcpyHostToDevice, st));
    }
  }
  const uint8_t* ph[3] = {in_h[0].as<uint8_t>(), in_h[1].as<uint8_t>(), in_h[2].as<uint8_t>()};
  const uint8_t* pm[3] = {in_m[0].as<uint8_t>(), in_m[1].as<uint8_t>(), in_m[2].as<uint8_t>()};
  const uint64_t match_words = 2 * W + 4;  // + padding for the OR tree's 64-bit funnel reads
  for (int p = 0; p < 3; ++p) {
    if (c->match[p].ensure(match_words * 4)) return fail(c, IRISMPC_GPU_ERR_DEVICE, "oom (match)");
    CK(c, cudaMemsetAsync(c->match[p].p, 0, match_words * 4, st));
  }
  const uint64_t nparty_m = vw.km ? 3 : 1;
  if (!or_only) {
    if (c->dots.ensure(3 * n * hb + nparty_m * n * mb + 64)) return fail(c, IRISMPC_GPU_ERR_DEVICE, "oom (components)");
    uint8_t* comp_h = c->dots.as<uint8_t>();
    uint8_t* comp_m = comp_h + round_up(3 * n * hb, 16);
    launch_parse_lane_shares(ph, n, hw, comp_h, bad.as<int>(), st);
    launch_parse_lane_shares(pm, n, vw.km ? mw : 8, comp_m, bad.as<int>(), st);
  } else {
    // component words straight into the match buffers (2 u32 per 64-lane word)
    Buf tmp;
    if (tmp.ensure(3 * 2 * W * 4 + 16)) return fail(c, IRISMPC_GPU_ERR_DEVICE, "oom");
    launch_parse_bit_shares(ph, W, n, tmp.as<uint32_t>(), bad.as<int>(), st);
    for (int p = 0; p < 3; ++p)
      CK(c, cudaMemcpyAsync(c->match[p].p, tmp.as<uint32_t>() + p * 2 * W, 2 * W * 4, cudaMemcpyDeviceToDevice, st));
    CK(c, cudaStreamSynchronize(st));
    tmp.release();
  }
  launches += or_only ? 1 : 2;
  CK(c, cudaGetLastError());
  {
    int h = 0;
    CK(c, cudaMemcpyAsync(&h, bad.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(c, cudaStreamSynchronize(st));
    if (h) return fail(c, IRISMPC_GPU_ERR_INCONSISTENT, "replicated share cross-check failed (bench payload)");
  }
  CK(c, cudaEventRecord(c->ev[1], st));

  const uint32_t nlift = V == kMpcLift ? 64u : 0u;
  const uint32_t ngates = nlift + 2u * vw.kc - 3u;
  auto seg_tasks = [](uint64_t lb, uint64_t le) { return (le - 1) / 1024 - lb / 1024 + 1; };
  const uint64_t kJob = 1ull << 24;
  const uint64_t njobs = or_only ? 0 : ceil_div(n, kJob);
  uint64_t total_slots = 0;
  ThrArgs ta{};
  ta.variant = V;
  ta.n = n;
  ta.W = W;
  ta.no_reshare = 1;
  ta.tile_kernels = 1;  // no GEMM beside it: the faster standalone kernels
  for (int k = 0; k < 3; ++k) {
    ta.pos[k] = c->pos[k];
    ta.key[k] = c->keys[k];
    const uint64_t inj = V == kMpcLift ? 64 * W + (k == 0 ? 2 * n : (k == 1 ? 0 : 6 * n)) : 0;
    ta.lift_base[k] = c->pos[k];
    ta.inj_base[k] = c->pos[k] + 64 * W;
    ta.msb_base[k] = c->pos[k] + inj;
  }
  ta.nlift = nlift;
  ta.ngates = ngates;
  ta.a = c->cfg.a;
  ta.b = c->cfg.b;
  ta.coef = 1.0 - 2.0 * c->cfg.match_ratio;
  const uint64_t octr = ++c->or_ctr;
  c->query_id++;
  c->last_groups = 0;  // the AGG tap is valid only after this call's share-exact OR tree
  ta.or_stream = or_stream_id(octr, c->cfg.shard_rank, 1);
  for (int p = 0; p < 3; ++p) ta.match[p] = c->match[p].as<uint32_t>();
  ta.match_w0 = 0;
  if (njobs) {
    if (ensure_host_segs(c, njobs + 1)) return IRISMPC_GPU_ERR_DEVICE;
    if (c->segs.ensure((njobs + 1) * sizeof(Seg))) return fail(c, IRISMPC_GPU_ERR_DEVICE, "oom (segs)");
    uint64_t max_g = 0, max_t = 0;
    for (uint64_t j = 0; j < njobs; ++j) {
      Seg& sg = c->h_segs_pinned[j];
      sg = Seg{};
      sg.lane_begin = j * kJob;
      sg.lane_end = std::min<uint64_t>(n, (j + 1) * kJob);
      sg.src = 0;
      sg.task_begin = 0;
      sg.q_first = sg.lane_begin / 1024;
      sg.w_first = sg.lane_begin / 64;
      sg.g_off = 0;
      sg.grp_begin = 0;
      sg.gblk_begin = 0;
      sg.slot = -1;  // the OR tree reads the match words
      const uint64_t nw = (sg.lane_end - 1) / 64 - sg.w_first + 1;
      total_slots += seg_tasks(sg.lane_begin, sg.lane_end);
      max_g = std::max<uint64_t>(max_g, 3ull * ngates * gate_row_words(nw));
      max_t = std::max<uint64_t>(max_t, seg_tasks(sg.lane_begin, sg.lane_end));
    }
    CK(c, cudaMemcpyAsync(c->segs.p, c->h_segs_pinned, njobs * sizeof(Seg), cudaMemcpyHostToDevice, st));
    const uint64_t cs = round_up(kJob, 8);
    if (c->ml_rs.ensure((V == kMpcLift ? 3 * cs * sizeof(uint16_t) : 0) + 16) ||
        c->diff.ensure(3 * cs * sizeof(uint32_t) + 16) || c->gate.ensure(max_g * sizeof(uint64_t) + 16) ||
        c->bits.ensure((V == kMpcLift ? 6 * max_t * 32 * sizeof(uint32_t) : 0) + 16) ||
        c->partial.ensure(3 * total_slots + 16))
      return fail(c, IRISMPC_GPU_ERR_DEVICE, "oom (threshold work buffers)");
    ta.ml_rs = c->ml_rs.as<uint16_t>();
    ta.diff = c->diff.as<uint32_t>();
    ta.cstride = cs;
    ta.gate = c->gate.as<uint64_t>();
    ta.bits = c->bits.as<uint32_t>();
    ta.partial = c->partial.as<uint8_t>();
    ta.nslots = total_slots;
    uint8_t* comp_h = c->dots.as<uint8_t>();
    uint8_t* comp_m = comp_h + round_up(3 * n * hb, 16);
    uint64_t task_off = 0;
    for (uint64_t j = 0; j < njobs; ++j) {
      const Seg& sg = c->h_segs_pinned[j];
      const uint64_t nl = sg.lane_end - sg.lane_begin;
      const uint64_t nw = (sg.lane_end - 1) / 64 - sg.w_first + 1;
      ThrArgs t = ta;
      t.segs = c->segs.as<Seg>() + j;
      t.nsegs = 1;
      t.ntasks = seg_tasks(sg.lane_begin, sg.lane_end);
      t.ngrp = (sg.lane_end - 1) / 8 - sg.lane_begin / 8 + 1;
      t.ngblk = 3ull * ngates * (nw / 8 + 2);
      t.ks_seg_threads = (uint32_t)t.ngblk;
      t.grp_seg_max = (uint32_t)t.ngrp;
      t.task_seg_max = (uint32_t)t.ntasks;
      t.nbits = t.ntasks * 32;
      t.or_elem_base = task_off * 64;
      task_off += t.ntasks;
      for (int p = 0; p < 3; ++p) {
        t.hd[p] = comp_h + (p * n + sg.lane_begin) * hb;
        t.ml[p] = comp_m + ((vw.km ? p : 0) * n + sg.lane_begin) * mb;
      }
      (void)nl;
      launch_threshold(t, st);
      CK(c, cudaGetLastError());
      launches += V == kMpcLift ? 5 : 3;
    }
  }
  CK(c, cudaEventRecord(c->ev[3], st));
  const bool do_or = or_only || with_or;
  if (do_or) {
    // or_tree over every lane (engine.cpp:508-512, 527-530): one group, the
    // reference's halving tree and draws (share-exact), then the open at P1
    if (c->person_out.ensure(3 + 16) || c->open_out.ensure(16))
      return fail(c, IRISMPC_GPU_ERR_DEVICE, "oom (or buffers)");
    OrTreeArgs oa{};
    for (int p = 0; p < 3; ++p) oa.match[p] = c->match[p].as<uint64_t>();
    oa.ngroups = 1;
    oa.db_lanes = n;
    oa.lanes = n;
    for (int k = 0; k < 3; ++k) oa.key[k] = c->keys[k];
    uint64_t rs[3];
    for (int k = 0; k < 3; ++k) rs[k] = or_only ? c->pos[k] : ta.msb_base[k] + (uint64_t)(2 * vw.kc - 3) * W;
    const uint64_t words = ortree_scratch_words(1, n);
    if (c->or_scr[0].ensure(words * 8) || c->or_scr[1].ensure(words * 8))
      return fail(c, IRISMPC_GPU_ERR_DEVICE, "oom (or tree)");
    uint64_t* scr[2] = {c->or_scr[0].as<uint64_t>(), c->or_scr[1].as<uint64_t>()};
    launches += launch_ortree(oa, rs, scr, c->person_out.as<uint8_t>(), st);
    c->last_groups = 1;
    launch_or_open(c->person_out.as<uint8_t>(), 1, 1, c->keys, or_stream_id(octr, c->cfg.shard_rank, 3),
                   c->open_out.as<uint8_t>(), st);
    CK(c, cudaGetLastError());
    launches += 1;
    if (opened_out) CK(c, cudaMemcpyAsync(opened_out, c->open_out.p, 1, cudaMemcpyDeviceToHost, st));
  }
  CK(c, cudaEventRecord(c->ev[4], st));
  if (lane_bits_out && !or_only) {
    std::vector<uint32_t> w[3];
    const uint64_t nw = ceil_div(n, 32);
    for (int p = 0; p < 3; ++p) {
      w[p].resize(nw);
      CK(c, cudaMemcpyAsync(w[p].data(), c->match[p].p, nw * 4, cudaMemcpyDeviceToHost, st));
    }
    CK(c, cudaStreamSynchronize(st));
    for (uint64_t i = 0; i < n; ++i)
      lane_bits_out[i] = (uint8_t)(((w[0][i / 32] ^ w[1][i / 32] ^ w[2][i / 32]) >> (i % 32)) & 1u);
  }
  CK(c, cudaStreamSynchronize(st));
  for (int p = 0; p < 3; ++p) {
    in_h[p].release();
    in_m[p].release();
  }
  bad.release();
  // advance the streams as the reference's comparison / or-tree call does
  uint64_t or_rounds = 0, or_bytes = 0;
  const uint64_t ord = do_or ? ref_or_draws(1, n, &or_rounds, &or_bytes) : 0;
  const uint64_t msb_draws = or_only ? 0 : (uint64_t)(2 * vw.kc - 3) * W;
  for (int k = 0; k < 3; ++k) c->pos[k] = (or_only ? c->pos[k] : ta.msb_base[k] + msb_draws) + ord;
  if (stats) {
    std::memset(stats, 0, sizeof(*stats));
    stats->batch = 1;
    stats->lanes = n;
    const uint64_t nb8 = ceil_div(n, 8);
    for (int p = 0; p < 3; ++p) {
      if (!or_only) {
        stats->lift_bytes[p] = V == kMpcLift ? 64 * nb8 + (p == 0 ? 8 * n : 4 * n) : 0;
        stats->msb_bytes[p] = (uint64_t)(2 * vw.kc - 3) * nb8;
      }
      stats->or_tree_bytes[p] = do_or ? or_bytes + (p == 0 ? 0 : 1) : 0;
    }
    stats->lift_rounds = (!or_only && V == kMpcLift) ? 21 : 0;
    stats->msb_rounds = or_only ? 0 : (uint64_t)vw.kc - 1;
    stats->or_tree_rounds = do_or ? or_rounds + 1 : 0;
    float ms = 0;
    cudaEventElapsedTime(&ms, c->ev[0], c->ev[4]);
    stats->wall_ms = ms;
    cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]);
    stats->prep_ms = ms;
    cudaEventElapsedTime(&ms, c->ev[1], c->ev[3]);
    stats->threshold_ms = ms;
    cudaEventElapsedTime(&ms, c->ev[3], c->ev[4]);
    stats->or_ms = ms;
    stats->kernel_launches = launches;
  }
  return 0;
}

}  // namespace

// =========================================================================== ABI

extern "C" {

int irismpc_gpu_seeds_from_master(uint64_t master, uint8_t out[48]) {
  uint8_t s[16], d[16];
  host_seed_from_u64(master, s);
  host_derive(s, 0x5eed, d);
  // Rng(d): 48 draws, one byte (low) each (deal_seeds, rep3.hpp:116-122)
  for (int i = 0; i < 48; ++i) {
    uint32_t blk[16];
    host_block(d, (uint64_t)i / 8, 0, blk);
    out[i] = (uint8_t)blk[2 * (i % 8)];
  }
  return 0;
}

size_t irismpc_gpu_record_bytes(uint32_t backend, uint32_t variant, uint32_t l) {
  if (variant > IRISMPC_GPU_VARIANT_NO_LIFT || backend > 1) return 0;
  return record_bytes(backend, variant, l);
}

uint64_t irismpc_gpu_lane_count(uint32_t persons, uint64_t s, uint32_t rotations, int membership) {
  if (membership) return s;
  return 2ull * persons * rotations * s + (uint64_t)persons * (persons ? persons - 1 : 0) / 2 * 4 * rotations;
}

int irismpc_gpu_create(const irismpc_gpu_config* cfg, irismpc_gpu_ctx** out) {
  if (!cfg || !out) return IRISMPC_GPU_ERR_CONFIG;
  *out = nullptr;
  std::string why;
  int rc = validate(cfg, &why);
  if (rc) {
    std::fprintf(stderr, "irismpc_gpu_create: %s\n", why.c_str());
    return rc;
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= cfg->device || cfg->device < 0) {
    std::fprintf(stderr, "irismpc_gpu_create: no CUDA device %d\n", cfg->device);
    return IRISMPC_GPU_ERR_DEVICE;
  }
  if (cudaSetDevice(cfg->device) != cudaSuccess) return IRISMPC_GPU_ERR_DEVICE;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, cfg->device) != cudaSuccess || prop.major != 10) {
    std::fprintf(stderr, "irismpc_gpu_create: device is not sm_100 (B200)\n");
    return IRISMPC_GPU_ERR_DEVICE;
  }
  auto* c = new irismpc_gpu_ctx;
  c->cfg = *cfg;
  c->shamir = cfg->backend == IRISMPC_GPU_BACKEND_SHAMIR;
  c->variant = (int)cfg->variant;
  c->vw = variant_widths(c->variant);
  c->l = cfg->l;
  c->l_pad = (uint32_t)round_up(cfg->l, kGemmBK);
  c->rec = record_bytes(cfg->backend, cfg->variant, cfg->l);
  {
    const uint64_t code_b = field_bytes(cfg->backend, c->vw.kh, cfg->l);
    const int widths[2] = {c->vw.kh / 8, c->vw.km / 8};
    for (int fi = 0; fi < 2; ++fi) {
      FieldPlanes& f = c->fld[fi];
      f.fmt.rec_bytes = c->rec;
      f.fmt.off = fi == 0 ? 0 : code_b;
      f.fmt.width = widths[fi];
      f.fmt.limbs = widths[fi] == 0 ? 1 : widths[fi];
      f.nparty = widths[fi] == 0 ? 1 : 3;
      f.nseg = (widths[fi] != 0 && !c->shamir) ? 2 : 1;
      f.out_bytes = f.fmt.limbs == 4 ? 4 : 2;
      // rotation-pair layout (and, with it, the Winograd rotation-pair GEMM) for integer
      // fields of rotated queries; IRISMPC_RP=0 keeps the natural K order, IRISMPC_RP=layout
      // the RP planes without the S planes (the large-DB fallback, for tests)
      static const bool rp_env = [] {
        const char* e = std::getenv("IRISMPC_RP");
        return !(e && e[0] == '0');
      }();
      f.fmt.rp = (rp_env && widths[fi] != 0 && cfg->rotations >= 3 && c->l_pad == cfg->l &&
                  rp_layout_ok(cfg->l, c->shamir)) ? 1 : 0;
    }
  }
  for (int k = 0; k < 3; ++k) c->keys[k] = key_of(cfg->seeds + 16 * k);
  // The threshold stream (st2) gets the higher priority: the threshold chain is
  // the critical path, and when both kernels want an SM the block scheduler
  // should seat the ALU-bound threshold blocks first and let the persistent
  // tensor-core GEMM fill in (measured +6% over the reverse at configs[1]).
  int prio_lo = 0, prio_hi = 0;
  cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
  if (const char* e = std::getenv("IRISMPC_PRIO_SWAP"); e && e[0] == '1') std::swap(prio_lo, prio_hi);
  if (cudaStreamCreateWithPriority(&c->st, cudaStreamNonBlocking, prio_lo) != cudaSuccess ||
      cudaStreamCreateWithPriority(&c->st2, cudaStreamNonBlocking, prio_hi) != cudaSuccess ||
      cudaStreamCreateWithPriority(&c->st3, cudaStreamNonBlocking, prio_hi) != cudaSuccess) {
    delete c;
    return IRISMPC_GPU_ERR_DEVICE;
  }
  for (auto& e : c->ev) cudaEventCreate(&e);
  uint32_t lam[6];
  lambdas(lam);
  set_lambda(lam);
  *out = c;
  return 0;
}

void irismpc_gpu_destroy(irismpc_gpu_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->cfg.device);
  cudaStreamSynchronize(c->st);
  drain(c);
  for (auto& q : c->qs) {
    Buf* qb[] = {&q.segs, &q.slot_begin, &q.match[0], &q.match[1], &q.match[2], &q.pair_dots, &q.open_out,
                 &q.qpay[0], &q.qpay[1], &q.qpay[2], &q.part, &q.all};
    for (Buf* b : qb) b->release();
    if (q.h_segs) cudaFreeHost(q.h_segs);
    if (q.h_match) cudaFreeHost(q.h_match);
    for (auto& e : q.ev)
      if (e) cudaEventDestroy(e);
    if (q.done) cudaEventDestroy(q.done);
    for (auto& e : q.gev) cudaEventDestroy(e);
  }
  for (auto& e : c->half_free)
    if (e) cudaEventDestroy(e);
  for (int k = 0; k < 2; ++k) {
    if (c->front_done[k]) cudaEventDestroy(c->front_done[k]);
    if (c->back_done[k]) cudaEventDestroy(c->back_done[k]);
    c->wk_ml_rs[k].release();
    c->wk_diff[k].release();
    c->wk_gate[k].release();
    c->wk_bits[k].release();
  }
  c->shard_nccl = nullptr;
  c->shard.reset();
  c->shard_part.release();
  c->shard_all.release();
  Buf* bufs[] = {&c->q_pay[0], &c->q_pay[1], &c->q_pay[2], &c->dots, &c->pair_dots, &c->segs, &c->partial,
                 &c->slot_begin, &c->person_out, &c->match[0], &c->match[1], &c->match[2], &c->open_out,
                 &c->ml_rs, &c->diff, &c->gate, &c->bits, &c->or_scr[0], &c->or_scr[1]};
  for (Buf* b : bufs) b->release();
  for (auto& f : c->fld) f.release();
  for (auto& t : c->tap_buf) t.release();
  c->tap_rows_dev.release();
  if (c->h_segs_pinned) cudaFreeHost(c->h_segs_pinned);
  for (auto& e : c->ev) cudaEventDestroy(e);
  for (auto& e : c->evg) cudaEventDestroy(e);
  for (auto& e : c->evt) cudaEventDestroy(e);
  cudaStreamSynchronize(c->st2);
  cudaStreamSynchronize(c->st3);
  cudaStreamDestroy(c->st2);
  cudaStreamDestroy(c->st3);
  cudaStreamDestroy(c->st);
  delete c;
}

const char* irismpc_gpu_last_error(const irismpc_gpu_ctx* c) { return c ? c->err.c_str() : "null context"; }

void* irismpc_gpu_stream(irismpc_gpu_ctx* c) { return c ? (void*)c->st : nullptr; }

int irismpc_gpu_load_db(irismpc_gpu_ctx* c, const uint8_t* const payload[3], const size_t len[3], uint64_t s) {
  if (!c) return IRISMPC_GPU_ERR_CONFIG;
  const Range nvtx_range("irismpc.load_db");
  cudaSetDevice(c->cfg.device);
  const size_t rec = c->rec;
  for (int p = 0; p < 3; ++p)
    if (len[p] != s * rec) return fail(c, IRISMPC_GPU_ERR_CONFIG, "db payload size mismatch");
  int rc = alloc_planes(c, s);
  if (rc) return rc;
  const uint64_t chunk = std::max<uint64_t>(1, (256ull << 20) / rec);
  Buf stage[3], bad;
  for (int p = 0; p < 3; ++p)
    if (stage[p].ensure(std::min<uint64_t>(chunk, s ? s : 1) * rec))
      return fail(c, IRISMPC_GPU_ERR_DEVICE, "oom (load staging)");
  if (bad.ensure(sizeof(int))) return fail(c, IRISMPC_GPU_ERR_DEVICE, "oom");
  CK(c, cudaMemsetAsync(bad.p, 0, sizeof(int), c->st));
  for (uint64_t r0 = 0; r0 < s; r0 += chunk) {
    const uint64_t nr = std::min<uint64_t>(chunk, s - r0);
    for (int p = 0; p < 3; ++p)
      CK(c, cudaMemcpyAsync(stage[p].p, payload[p] + r0 * rec, nr * rec, cudaMemcpyHostToDevice, c->st));
    const uint8_t* dp[3] = {stage[0].as<uint8_t>(), stage[1].as<uint8_t>(), stage[2].as<uint8_t>()};
    rc = parse_rows(c, dp, nr, r0, &bad);
    if (rc) return rc;
    CK(c, cudaStreamSynchronize(c->st));
  }
  rc = finish_load(c, c->shamir ? nullptr : &bad);
  for (auto& b : stage) b.release();
  bad.release();
  return rc;
}

int irismpc_gpu_load_db_device(irismpc_gpu_ctx* c, const uint8_t* const dpayload[3], const size_t len[3],
                               uint64_t s) {
  if (!c) return IRISMPC_GPU_ERR_CONFIG;
  const Range nvtx_range("irismpc.load_db_device");
  cudaSetDevice(c->cfg.device);
  const size_t rec = c->rec;
  for (int p = 0; p < 3; ++p)
    if (len[p] != s * rec) return fail(c, IRISMPC_GPU_ERR_CONFIG, "db payload size mismatch");
  int rc = alloc_planes(c, s);
  if (rc) return rc;
  Buf bad;
  if (bad.ensure(sizeof(int))) return fail(c, IRISMPC_GPU_ERR_DEVICE, "oom");
  CK(c, cudaMemsetAsync(bad.p, 0, sizeof(int), c->st));
  rc = parse_rows(c, dpayload, s, 0, &bad);
  if (rc) return rc;
  rc = finish_load(c, c->shamir ? nullptr : &bad);
  bad.release();
  return rc;
}

int irismpc_gpu_load_db_files(irismpc_gpu_ctx* c, const char* const paths[3]) {
  if (!c || !paths) return IRISMPC_GPU_ERR_CONFIG;
  const Range nvtx_range("irismpc.load_db_files");
  cudaSetDevice(c->cfg.device);
  irismpc_gpu_share_header h[3];
  for (int p = 0; p < 3; ++p) {
    if (irismpc_gpu_read_share_header(paths[p], &h[p]))
      return fail(c, IRISMPC_GPU_ERR_CONFIG, std::string("not a valid IRS1 share file: ") + (paths[p] ? paths[p] : "(null)"));
    if (h[p].party != (uint32_t)(p + 1)) return fail(c, IRISMPC_GPU_ERR_CONFIG, "share file belongs to another party");
    if (h[p].backend != c->cfg.backend || h[p].variant != c->cfg.variant || h[p].l != c->l)
      return fail(c, IRISMPC_GPU_ERR_CONFIG, "share file does not match config");
    if (h[p].s != h[0].s) return fail(c, IRISMPC_GPU_ERR_CONFIG, "share files disagree on s");
  }
  const uint64_t s = h[0].s, rec = c->rec;
  int rc = alloc_planes(c, s);
  if (rc) return rc;
  FILE* f[3] = {nullptr, nullptr, nullptr};
  auto close_all = [&] {
    for (auto& x : f)
      if (x) std::fclose(x);
  };
  for (int p = 0; p < 3; ++p) {
    f[p] = std::fopen(paths[p], "rb");
    if (!f[p] || std::fseek(f[p], 24, SEEK_SET) != 0) {
      close_all();
      return fail(c, IRISMPC_GPU_ERR_CONFIG, "cannot open share file");
    }
  }
  // two pinned slots: the disk read of chunk i+1 overlaps the H2D + parse of chunk i
  const uint64_t chunk = std::max<uint64_t>(1, std::min<uint64_t>(s ? s : 1, (128ull << 20) / rec));
  uint8_t* host[2] = {nullptr, nullptr};
  Buf dev[2], bad;
  cudaEvent_t done[2] = {nullptr, nullptr};
  int status = 0;
  for (int k = 0; k < 2 && !status; ++k) {
    if (cudaMallocHost(&host[k], 3 * chunk * rec) != cudaSuccess || dev[k].ensure(3 * chunk * rec) ||
        cudaEventCreateWithFlags(&done[k], cudaEventDisableTiming) != cudaSuccess)
      status = fail(c, IRISMPC_GPU_ERR_DEVICE, "oom (file load staging)");
  }
  if (!status && (bad.ensure(sizeof(int)) || cudaMemsetAsync(bad.p, 0, sizeof(int), c->st) != cudaSuccess))
    status = fail(c, IRISMPC_GPU_ERR_DEVICE, "oom");
  for (uint64_t r0 = 0, i = 0; r0 < s && !status; r0 += chunk, ++i) {
    const int k = (int)(i % 2);
    const uint64_t nr = std::min<uint64_t>(chunk, s - r0);
    if (i >= 2 && cudaEventSynchronize(done[k]) != cudaSuccess) {
      status = fail(c, IRISMPC_GPU_ERR_DEVICE, "file load: device fault");
      break;
    }
    for (int p = 0; p < 3 && !status; ++p)
      if (std::fread(host[k] + p * chunk * rec, 1, nr * rec, f[p]) != nr * rec)
        status = fail(c, IRISMPC_GPU_ERR_CONFIG, "short read: share file");
    if (status) break;
    const uint8_t* dp[3];
    for (int p = 0; p < 3; ++p) {
      dp[p] = dev[k].as<uint8_t>() + p * chunk * rec;
      if (cudaMemcpyAsync(const_cast<uint8_t*>(dp[p]), host[k] + p * chunk * rec, nr * rec, cudaMemcpyHostToDevice,
                          c->st) != cudaSuccess)
        status = fail(c, IRISMPC_GPU_ERR_DEVICE, "file load: H2D failed");
    }
    if (status) break;
    status = parse_rows(c, dp, nr, r0, c->shamir ? nullptr : &bad);
    if (!status && cudaEventRecord(done[k], c->st) != cudaSuccess)
      status = fail(c, IRISMPC_GPU_ERR_DEVICE, "file load: event");
  }
  close_all();
  if (!status) status = finish_load(c, c->shamir ? nullptr : &bad);
  cudaStreamSynchronize(c->st);
  for (int k = 0; k < 2; ++k) {
    if (host[k]) cudaFreeHost(host[k]);
    if (done[k]) cudaEventDestroy(done[k]);
    dev[k].release();
  }
  bad.release();
  return status;
}

int irismpc_gpu_batch_query(irismpc_gpu_ctx* c, const uint8_t* const q[3], const size_t qlen[3], uint32_t persons,
                            uint8_t* person_match_out, uint8_t* row_bits_out, irismpc_gpu_stats* stats) {
  if (!c) return IRISMPC_GPU_ERR_CONFIG;
  const Range nvtx_range("irismpc.batch_query");
  cudaSetDevice(c->cfg.device);
  const uint8_t* none[3] = {nullptr, nullptr, nullptr};
  return run_query(c, none, qlen, persons, 0, 0, person_match_out, row_bits_out, nullptr, stats, true, q);
}

int irismpc_gpu_batch_query_device(irismpc_gpu_ctx* c, const uint8_t* const dq[3], const size_t qlen[3],
                                   uint32_t persons, uint8_t* person_match_out, uint8_t* row_bits_out,
                                   irismpc_gpu_stats* stats) {
  if (!c) return IRISMPC_GPU_ERR_CONFIG;
  const Range nvtx_range("irismpc.batch_query_device");
  cudaSetDevice(c->cfg.device);
  return run_query(c, dq, qlen, persons, 0, 0, person_match_out, row_bits_out, nullptr, stats, false, nullptr);
}

int irismpc_gpu_membership(irismpc_gpu_ctx* c, const uint8_t* const q[3], const size_t qlen[3], uint8_t* match_out,
                           uint8_t* row_bits_out, irismpc_gpu_stats* stats) {
  if (!c) return IRISMPC_GPU_ERR_CONFIG;
  const Range nvtx_range("irismpc.membership");
  cudaSetDevice(c->cfg.device);
  const uint8_t* none[3] = {nullptr, nullptr, nullptr};
  return run_query(c, none, qlen, 1, 1, 0, match_out, row_bits_out, nullptr, stats, true, q);
}

int irismpc_gpu_batch_query_submit(irismpc_gpu_ctx* c, const uint8_t* const dq[3], const size_t qlen[3],
                                   uint32_t persons, uint8_t* person_match_out, uint64_t* ticket) {
  if (!c || !ticket) return IRISMPC_GPU_ERR_CONFIG;
  const Range nvtx_range("irismpc.batch_query_submit");
  cudaSetDevice(c->cfg.device);
  if (c->taps || c->tap_k || c->cfg.debug_rows)
    return fail(c, IRISMPC_GPU_ERR_CONFIG, "streaming queries run without taps / debug_rows");
  return run_query(c, dq, qlen, persons, 0, 0, person_match_out, nullptr, nullptr, nullptr, false, nullptr, ticket);
}

int irismpc_gpu_batch_query_wait(irismpc_gpu_ctx* c, uint64_t ticket, irismpc_gpu_stats* stats) {
  if (!c) return IRISMPC_GPU_ERR_CONFIG;
  const Range nvtx_range("irismpc.batch_query_wait");
  cudaSetDevice(c->cfg.device);
  for (auto& q : c->qs) {
    if (q.ticket != ticket) continue;
    if (q.inflight) {
      const int rc = finish_slot(c, q);
      if (rc) return rc;
    }
    if (stats) *stats = q.stats;
    return 0;
  }
  return fail(c, IRISMPC_GPU_ERR_CONFIG, "unknown or expired ticket (wait for a ticket before submitting two more)");
}

int irismpc_gpu_batch_query_partial(irismpc_gpu_ctx* c, const uint8_t* const dq[3], const size_t qlen[3],
                                    uint32_t persons, uint8_t* partial_out_dev, irismpc_gpu_stats* stats) {
  if (!c) return IRISMPC_GPU_ERR_CONFIG;
  const Range nvtx_range("irismpc.batch_query_partial");
  cudaSetDevice(c->cfg.device);
  return run_query(c, dq, qlen, persons, 0, 1, nullptr, nullptr, partial_out_dev, stats, false, nullptr);
}

int irismpc_gpu_or_open(irismpc_gpu_ctx* c, const uint8_t* partials_dev, uint32_t G, uint32_t persons,
                        uint8_t* person_match_out) {
  if (!c) return IRISMPC_GPU_ERR_CONFIG;
  cudaSetDevice(c->cfg.device);
  if (c->open_out.ensure(persons + 16)) return fail(c, IRISMPC_GPU_ERR_DEVICE, "oom");
  // the partial query advanced or_ctr; the cross-shard OR + open draws that query's kind-3 stream
  launch_or_open(partials_dev, G, persons, c->keys, or_stream_id(c->or_ctr, c->cfg.shard_rank, 3),
                 c->open_out.as<uint8_t>(), c->st);
  CK(c, cudaGetLastError());
  CK(c, cudaMemcpyAsync(person_match_out, c->open_out.p, persons, cudaMemcpyDeviceToHost, c->st));
  CK(c, cudaStreamSynchronize(c->st));
  return 0;
}

int irismpc_gpu_comparison_only(irismpc_gpu_ctx* c, const uint8_t* const hd_payload[3], const size_t hd_len[3],
                                const uint8_t* const ml_payload[3], const size_t ml_len[3], uint64_t lanes,
                                int with_or_tree, uint8_t* opened_out, uint8_t* lane_bits_out,
                                irismpc_gpu_stats* stats) {
  if (!c || !hd_payload || !ml_payload) return IRISMPC_GPU_ERR_CONFIG;
  const Range nvtx_range("irismpc.comparison_only");
  cudaSetDevice(c->cfg.device);
  if (lanes == 0) return fail(c, IRISMPC_GPU_ERR_CONFIG, "no lanes");
  return run_compare(c, 0, hd_payload, hd_len, ml_payload, ml_len, lanes, with_or_tree, opened_out, lane_bits_out,
                     stats);
}

int irismpc_gpu_or_tree_only(irismpc_gpu_ctx* c, const uint8_t* const payload[3], const size_t len[3],
                             uint64_t lanes, uint8_t* opened_out, irismpc_gpu_stats* stats) {
  if (!c || !payload) return IRISMPC_GPU_ERR_CONFIG;
  const Range nvtx_range("irismpc.or_tree_only");
  cudaSetDevice(c->cfg.device);
  if (lanes == 0) return fail(c, IRISMPC_GPU_ERR_CONFIG, "no lanes");
  return run_compare(c, 1, payload, len, nullptr, nullptr, lanes, 1, opened_out, nullptr, stats);
}

int irismpc_gpu_shard_group_create(uint32_t world, irismpc_gpu_shard_group** out) {
  if (!out || world == 0) return IRISMPC_GPU_ERR_CONFIG;
  auto* g = new irismpc_gpu_shard_group;
  g->world = world;
  g->ptr.assign(world, nullptr);
  *out = g;
  return 0;
}

void irismpc_gpu_shard_group_destroy(irismpc_gpu_shard_group* g) { delete g; }

static int shard_check(irismpc_gpu_ctx* c, uint32_t world) {
  if (c->cfg.shard_rank >= world) return fail(c, IRISMPC_GPU_ERR_CONFIG, "shard_rank >= world size");
  if (world > 1 && c->cfg.db_rows_total == 0)
    return fail(c, IRISMPC_GPU_ERR_CONFIG, "a sharded context needs db_rows_total (the whole DB's rows)");
  return 0;
}

int irismpc_gpu_shard_attach_inproc(irismpc_gpu_ctx* c, irismpc_gpu_shard_group* g) {
  if (!c || !g) return IRISMPC_GPU_ERR_CONFIG;
  if (int rc = shard_check(c, g->world)) return rc;
  c->shard_nccl = nullptr;
  auto sc = std::make_unique<InprocShardComm>();
  sc->g = g;
  sc->world = g->world;
  sc->rank = c->cfg.shard_rank;
  c->shard = std::move(sc);
  return 0;
}

int irismpc_gpu_shard_attach_nccl(irismpc_gpu_ctx* c, const uint8_t nccl_id[128], uint32_t world) {
  if (!c || !nccl_id) return IRISMPC_GPU_ERR_CONFIG;
  if (int rc = shard_check(c, world)) return rc;
  if (!nccl().ok) return fail(c, IRISMPC_GPU_ERR_DEVICE, "libnccl could not be loaded");
  cudaSetDevice(c->cfg.device);
  auto sc = std::make_unique<NcclShardComm>();
  ncclUniqueId id;
  std::memcpy(&id, nccl_id, sizeof(id));
  const ncclResult_t r = nccl().comm_init_rank(&sc->comm, (int)world, id, (int)c->cfg.shard_rank);
  if (r != ncclSuccess) return fail(c, IRISMPC_GPU_ERR_DEVICE, std::string("ncclCommInitRank: ") + nccl().error_string(r));
  if (nccl().comm_split && nccl().comm_split(sc->comm, 0, (int)c->cfg.shard_rank, &sc->comm2, nullptr) != ncclSuccess)
    sc->comm2 = nullptr;  // streaming sharded queries then unavailable (synchronous ones still work)
  sc->world = world;
  sc->rank = c->cfg.shard_rank;
  c->shard_nccl = sc.get();
  c->shard = std::move(sc);
  return 0;
}

// One query over the row-sharded DB: broadcast of the query
// payloads from shard 0, this shard's query up to the per-person XOR-shared
// aggregate (never opened), gather of every shard's [3][groups] partial to
// shard 0, the MPC-OR across shards and the open at P1 there.
static int sharded_query(irismpc_gpu_ctx* c, const uint8_t* const q[3], const size_t qlen[3], uint32_t persons,
                         int membership, bool host_input, uint8_t* match_out, irismpc_gpu_stats* stats) {
  if (!c->shard) return fail(c, IRISMPC_GPU_ERR_CONFIG, "context is not attached to a shard group");
  ShardComm& sc = *c->shard;
  const uint32_t groups = membership ? 1u : persons;
  const uint8_t* dq[3];
  for (int p = 0; p < 3; ++p) {
    if (c->q_pay[p].ensure(qlen[p] + 16)) return fail(c, IRISMPC_GPU_ERR_DEVICE, "oom (query payload)");
    if (sc.rank == 0) {
      if (!q || !q[p]) return fail(c, IRISMPC_GPU_ERR_CONFIG, "shard 0 needs the query payloads");
      if (host_input)
        CK(c, cudaMemcpyAsync(c->q_pay[p].p, q[p], qlen[p], cudaMemcpyHostToDevice, c->st));
      else if (q[p] != c->q_pay[p].as<uint8_t>())
        CK(c, cudaMemcpyAsync(c->q_pay[p].p, q[p], qlen[p], cudaMemcpyDeviceToDevice, c->st));
    }
  }
  for (int p = 0; p < 3; ++p) {  // (1) query-share broadcast
    const std::string e = sc.bcast(c->q_pay[p].p, qlen[p], c->st);
    if (!e.empty()) return fail(c, IRISMPC_GPU_ERR_DEVICE, e);
    dq[p] = c->q_pay[p].as<uint8_t>();
  }
  if (c->shard_part.ensure(3ull * groups + 16) || c->shard_all.ensure(3ull * groups * sc.world + 16))
    return fail(c, IRISMPC_GPU_ERR_DEVICE, "oom (shard partials)");
  const int rc = run_query(c, dq, qlen, persons, membership, 1, nullptr, nullptr, c->shard_part.as<uint8_t>(), stats,
                           false, nullptr);
  if (rc) return rc;
  const std::string e = sc.gather(c->shard_part.p, c->shard_all.p, 3ull * groups, c->st);  // (2)
  if (!e.empty()) return fail(c, IRISMPC_GPU_ERR_DEVICE, e);
  if (sc.rank == 0) {
    if (c->open_out.ensure(groups + 16)) return fail(c, IRISMPC_GPU_ERR_DEVICE, "oom");
    launch_or_open(c->shard_all.as<uint8_t>(), sc.world, groups, c->keys, or_stream_id(c->or_ctr, 0, 3),
                   c->open_out.as<uint8_t>(), c->st);
    CK(c, cudaGetLastError());
    if (match_out) CK(c, cudaMemcpyAsync(match_out, c->open_out.p, groups, cudaMemcpyDeviceToHost, c->st));
  }
  CK(c, cudaStreamSynchronize(c->st));
  if (stats) stats->kernel_launches += sc.rank == 0 ? 1 : 0;
  return 0;
}

// Streaming sharded query (NCCL only): everything is stream-ordered, no host sync --
// the query payloads are broadcast on the GEMM stream into this slot's buffers, the
// shard's query runs up to its partial, and the gather (second communicator), the
// cross-shard OR and the open follow on the threshold stream, so the GEMM stream of
// every shard runs into the next query like the single-GPU streaming path.
int irismpc_gpu_sharded_batch_query_submit(irismpc_gpu_ctx* c, const uint8_t* const dq[3], const size_t qlen[3],
                                           uint32_t persons, uint8_t* person_match_out, uint64_t* ticket) {
  if (!c || !ticket) return IRISMPC_GPU_ERR_CONFIG;
  const Range nvtx_range("irismpc.sharded_batch_query_submit");
  cudaSetDevice(c->cfg.device);
  NcclShardComm* nc = c->shard_nccl;
  if (!nc || !nc->comm2) return fail(c, IRISMPC_GPU_ERR_CONFIG, "streaming sharded queries need an NCCL shard attach");
  if (c->taps || c->tap_k || c->cfg.debug_rows)
    return fail(c, IRISMPC_GPU_ERR_CONFIG, "streaming queries run without taps / debug_rows");
  QSlot& Q = c->qs[c->par];  // the slot run_query takes next
  if (Q.inflight) {
    const int rc = finish_slot(c, Q);
    if (rc) return rc;
  }
  const uint32_t groups = persons;
  const uint8_t* qp[3];
  ncclResult_t r = nccl().group_start();
  for (int p = 0; p < 3 && r == ncclSuccess; ++p) {
    if (Q.qpay[p].ensure(qlen[p] + 16)) return fail(c, IRISMPC_GPU_ERR_DEVICE, "oom (query payload)");
    if (nc->rank == 0) {
      if (!dq || !dq[p]) return fail(c, IRISMPC_GPU_ERR_CONFIG, "shard 0 needs the query payloads");
      CK(c, cudaMemcpyAsync(Q.qpay[p].p, dq[p], qlen[p], cudaMemcpyDeviceToDevice, c->st));
    }
    r = nccl().broadcast(Q.qpay[p].p, Q.qpay[p].p, qlen[p], ncclUint8, 0, nc->comm, c->st);
    qp[p] = Q.qpay[p].as<uint8_t>();
  }
  const ncclResult_t r2 = nccl().group_end();
  if (r != ncclSuccess || r2 != ncclSuccess)
    return fail(c, IRISMPC_GPU_ERR_DEVICE, std::string("nccl broadcast: ") + nccl().error_string(r ? r : r2));
  if (Q.part.ensure(3ull * groups + 16) || Q.all.ensure(3ull * groups * nc->world + 16))
    return fail(c, IRISMPC_GPU_ERR_DEVICE, "oom (shard partials)");
  uint64_t t = 0;
  int rc = run_query(c, qp, qlen, persons, 0, 1, nullptr, nullptr, Q.part.as<uint8_t>(), nullptr, false, nullptr, &t);
  if (rc) return rc;
  // run_query queued the partial hand-off on the threshold stream of this slot; the rest follows it
  cudaStream_t st2 = c->serial ? c->st : c->st2;
  const ncclResult_t r3 = nccl().all_gather(Q.part.p, Q.all.p, 3ull * groups, ncclUint8, nc->comm2, st2);
  if (r3 != ncclSuccess) return fail(c, IRISMPC_GPU_ERR_DEVICE, std::string("nccl all_gather: ") + nccl().error_string(r3));
  if (nc->rank == 0) {
    if (Q.open_out.ensure(groups + 16)) return fail(c, IRISMPC_GPU_ERR_DEVICE, "oom");
    if (groups + 16 > Q.h_match_cap) {
      if (Q.h_match) cudaFreeHost(Q.h_match);
      Q.h_match = nullptr;
      Q.h_match_cap = 0;
      CK(c, cudaMallocHost(&Q.h_match, groups + 16));
      Q.h_match_cap = groups + 16;
    }
    launch_or_open(Q.all.as<uint8_t>(), nc->world, groups, c->keys, or_stream_id(c->or_ctr, 0, 3),
                   Q.open_out.as<uint8_t>(), st2);
    CK(c, cudaGetLastError());
    CK(c, cudaMemcpyAsync(Q.h_match, Q.open_out.p, groups, cudaMemcpyDeviceToHost, st2));
    Q.mode = 0;
    Q.match_out = person_match_out;
    Q.stats.kernel_launches += 1;
  }
  CK(c, cudaEventRecord(Q.ev[4], st2));
  CK(c, cudaEventRecord(Q.done, st2));
  *ticket = t;
  return 0;
}

int irismpc_gpu_sharded_batch_query(irismpc_gpu_ctx* c, const uint8_t* const q[3], const size_t qlen[3],
                                    uint32_t persons, uint8_t* person_match_out, irismpc_gpu_stats* stats) {
  if (!c) return IRISMPC_GPU_ERR_CONFIG;
  const Range nvtx_range("irismpc.sharded_batch_query");
  cudaSetDevice(c->cfg.device);
  return sharded_query(c, q, qlen, persons, 0, true, person_match_out, stats);
}

int irismpc_gpu_sharded_batch_query_device(irismpc_gpu_ctx* c, const uint8_t* const dq[3], const size_t qlen[3],
                                           uint32_t persons, uint8_t* person_match_out, irismpc_gpu_stats* stats) {
  if (!c) return IRISMPC_GPU_ERR_CONFIG;
  const Range nvtx_range("irismpc.sharded_batch_query_device");
  cudaSetDevice(c->cfg.device);
  return sharded_query(c, dq, qlen, persons, 0, false, person_match_out, stats);
}

int irismpc_gpu_sharded_membership(irismpc_gpu_ctx* c, const uint8_t* const q[3], const size_t qlen[3],
                                   uint8_t* match_out, irismpc_gpu_stats* stats) {
  if (!c) return IRISMPC_GPU_ERR_CONFIG;
  const Range nvtx_range("irismpc.sharded_membership");
  cudaSetDevice(c->cfg.device);
  return sharded_query(c, q, qlen, 1, 1, true, match_out, stats);
}

int irismpc_gpu_get_stream_positions(const irismpc_gpu_ctx* c, uint64_t pos[3]) {
  if (!c) return IRISMPC_GPU_ERR_CONFIG;
  for (int k = 0; k < 3; ++k) pos[k] = c->pos[k];
  return 0;
}

int irismpc_gpu_set_stream_positions(irismpc_gpu_ctx* c, const uint64_t pos[3]) {
  if (!c) return IRISMPC_GPU_ERR_CONFIG;
  for (int k = 0; k < 3; ++k) c->pos[k] = pos[k];
  return 0;
}

int irismpc_gpu_synth_records(irismpc_gpu_ctx* c, uint64_t rng_seed, uint64_t first, uint64_t count,
                              double mask_density, uint64_t* codes_dev, uint64_t* masks_dev) {
  if (!c) return IRISMPC_GPU_ERR_CONFIG;
  cudaSetDevice(c->cfg.device);
  uint8_t s[16];
  host_seed_from_u64(rng_seed, s);
  launch_synth_records(key_of(s), first, count, c->l, mask_density, codes_dev, masks_dev, c->st);
  CK(c, cudaGetLastError());
  CK(c, cudaStreamSynchronize(c->st));
  return 0;
}

int irismpc_gpu_deal_payload(irismpc_gpu_ctx* c, uint64_t deal_seed, uint64_t tag, uint64_t first_record,
                             uint64_t nrec, const uint64_t* codes_dev, const uint64_t* masks_dev,
                             uint8_t* const out_dev[3]) {
  if (!c) return IRISMPC_GPU_ERR_CONFIG;
  cudaSetDevice(c->cfg.device);
  uint8_t s[16], d[16];
  host_seed_from_u64(deal_seed, s);
  host_derive(s, tag, d);
  launch_deal(key_of(d), first_record, nrec, c->l, c->shamir, c->variant, codes_dev, masks_dev, out_dev[0],
              out_dev[1], out_dev[2], c->st);
  CK(c, cudaGetLastError());
  CK(c, cudaStreamSynchronize(c->st));
  return 0;
}

int irismpc_gpu_synth_db(irismpc_gpu_ctx* c, uint64_t s, uint64_t rng_seed, uint64_t first, double mask_density,
                         uint64_t deal_seed) {
  if (!c) return IRISMPC_GPU_ERR_CONFIG;
  const Range nvtx_range("irismpc.synth_db");
  cudaSetDevice(c->cfg.device);
  int rc = alloc_planes(c, s);
  if (rc) return rc;
  const size_t rec = c->rec;
  const uint64_t wl = (c->l + 63) / 64;
  const uint64_t chunk = std::max<uint64_t>(1, std::min<uint64_t>(s ? s : 1, (512ull << 20) / rec));
  Buf codes, masks, pay[3];
  if (codes.ensure(chunk * wl * 8) || masks.ensure(chunk * wl * 8)) return fail(c, IRISMPC_GPU_ERR_DEVICE, "oom");
  for (auto& p : pay)
    if (p.ensure(chunk * rec)) return fail(c, IRISMPC_GPU_ERR_DEVICE, "oom");
  uint8_t sr[16], sd[16], dd[16];
  host_seed_from_u64(rng_seed, sr);
  host_seed_from_u64(deal_seed, sd);
  host_derive(sd, 1, dd);
  for (uint64_t r0 = 0; r0 < s; r0 += chunk) {
    const uint64_t nr = std::min<uint64_t>(chunk, s - r0);
    launch_synth_records(key_of(sr), first + r0, nr, c->l, mask_density, codes.as<uint64_t>(),
                         masks.as<uint64_t>(), c->st);
    launch_deal(key_of(dd), first + r0, nr, c->l, c->shamir, c->variant, codes.as<uint64_t>(), masks.as<uint64_t>(),
                pay[0].as<uint8_t>(), pay[1].as<uint8_t>(), pay[2].as<uint8_t>(), c->st);
    const uint8_t* dp[3] = {pay[0].as<uint8_t>(), pay[1].as<uint8_t>(), pay[2].as<uint8_t>()};
    rc = parse_rows(c, dp, nr, r0, nullptr);
    if (rc) return rc;
  }
  CK(c, cudaGetLastError());
  rc = finish_load(c, nullptr);
  codes.release();
  masks.release();
  for (auto& p : pay) p.release();
  return rc;
}

int irismpc_gpu_profile(irismpc_gpu_ctx* c, int on) {
  if (!c) return IRISMPC_GPU_ERR_CONFIG;
  cudaSetDevice(c->cfg.device);
  if (int rc = drain(c)) return rc;
  c->serial = on != 0;
  prof_enable(on != 0);
  return 0;
}

int irismpc_gpu_threshold_kernels(irismpc_gpu_ctx* c, int tile) {
  if (!c) return IRISMPC_GPU_ERR_CONFIG;
  c->thr_tile = tile != 0;
  return 0;
}

int irismpc_gpu_profile_read(irismpc_gpu_ctx* c, char (*names)[48], double* ms, uint64_t* launches, uint32_t max,
                             uint32_t* count) {
  if (!c || !count) return IRISMPC_GPU_ERR_CONFIG;
  cudaSetDevice(c->cfg.device);
  *count = (uint32_t)prof_take(names, ms, launches, max);
  return 0;
}

int irismpc_gpu_tap_rows(irismpc_gpu_ctx* c, const uint64_t* rows, uint32_t k) {
  if (!c || (k && !rows)) return IRISMPC_GPU_ERR_CONFIG;
  cudaSetDevice(c->cfg.device);
  for (uint32_t i = 0; i < k; ++i)
    if (rows[i] >= c->s) return fail(c, IRISMPC_GPU_ERR_BOUNDS, "tap row outside this shard");
  c->tap_k = 0;
  if (k) {
    if (c->tap_rows_dev.ensure(k * sizeof(uint64_t))) return fail(c, IRISMPC_GPU_ERR_DEVICE, "oom (tap rows)");
    CK(c, cudaMemcpy(c->tap_rows_dev.p, rows, k * sizeof(uint64_t), cudaMemcpyHostToDevice));
  }
  c->tap_k = k;
  return 0;
}

int irismpc_gpu_enable_taps(irismpc_gpu_ctx* c, int enable) {
  if (!c) return IRISMPC_GPU_ERR_CONFIG;
  c->taps = enable != 0;
  return 0;
}

int irismpc_gpu_read_tap(irismpc_gpu_ctx* c, int tap, void* host_out, size_t bytes) {
  if (c && drain(c)) return IRISMPC_GPU_ERR_DEVICE;
  if (!c || tap < 1 || tap > 8) return IRISMPC_GPU_ERR_CONFIG;
  if (tap == 8) {  // the OR tree's output components, [3][groups] in person_out
    if (!c->person_out.p || bytes > 3ull * c->last_groups) return fail(c, IRISMPC_GPU_ERR_CONFIG, "no OR-tree output");
    cudaSetDevice(c->cfg.device);
    CK(c, cudaMemcpy(host_out, c->person_out.p, bytes, cudaMemcpyDeviceToHost));
    return 0;
  }
  if (!c->tap_buf[tap - 1].p) return fail(c, IRISMPC_GPU_ERR_CONFIG, "tap not captured");
  const size_t have = c->tap_bytes[tap - 1];
  if (bytes > have) return fail(c, IRISMPC_GPU_ERR_CONFIG, "tap read larger than captured");
  cudaSetDevice(c->cfg.device);
  CK(c, cudaMemcpy(host_out, c->tap_buf[tap - 1].p, bytes, cudaMemcpyDeviceToHost));
  return 0;
}

}  // extern "C"
