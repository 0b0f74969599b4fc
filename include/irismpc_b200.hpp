// irismpc_b200.hpp — header-only C++ host API over the C-ABI (irismpc_gpu.h),
// shaped like the reference library so existing callers drop in:
//
//   reference (/root/reference/proj)                      here
//   EngineConfig            engine.hpp:33-44        ->    irismpc_b200::EngineConfig
//   Session<B,16,16>        engine.hpp:225-275      ->    irismpc_b200::Session (all 3 parties, one GPU)
//   party_batch_query       engine.hpp:311-313      ->    irismpc_b200::ThreePartyGpu::party_batch_query
//   party_membership        engine.hpp:307-309      ->    irismpc_b200::ThreePartyGpu::party_membership
//   MembershipResult        engine.hpp:58-66        ->    irismpc_b200::MembershipResult
//   QueryStats              engine.hpp:46-56        ->    irismpc_b200::QueryStats
//   Error / BoundsError / TransportError / InconsistentShareError (errors.hpp:22-50)
//
// Per-party callers keep their three threads: each calls party_batch_query with
// its own payloads; the last one to arrive launches the fused 3-party GPU query
// and every caller returns its MembershipResult (person_match filled at P1, as
// kOutputParty = p1, engine.hpp:68).
#pragma once

#include <array>
#include <condition_variable>
#include <cstdint>
#include <memory>
#include <mutex>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "irismpc_gpu.h"

namespace irismpc_b200 {

struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct TransportError : Error {  // device failure: the in-process "transport" is the GPU
  using Error::Error;
};
struct BoundsError : Error {
  using Error::Error;
};
struct InconsistentShareError : Error {
  using Error::Error;
};

inline void check(int rc, const char* what, const irismpc_gpu_ctx* ctx = nullptr) {
  if (rc == IRISMPC_GPU_OK) return;
  std::string msg = std::string(what) + ": " + (ctx ? irismpc_gpu_last_error(ctx) : "");
  switch (rc) {
    case IRISMPC_GPU_ERR_BOUNDS: throw BoundsError(msg);
    case IRISMPC_GPU_ERR_DEVICE: throw TransportError(msg);
    case IRISMPC_GPU_ERR_INCONSISTENT: throw InconsistentShareError(msg);
    default: throw Error(msg);
  }
}

enum class Backend : std::uint8_t { replicated = 0, shamir = 1 };
enum class Variant : std::uint8_t { plain_mask = 0, mpc_lift = 1, const_lift = 2, no_lift = 3 };  // shares.hpp:28

inline const char* to_string(Variant v) {  // shares.cpp:22-33
  switch (v) {
    case Variant::plain_mask: return "plain-mask";
    case Variant::mpc_lift: return "mpc-lift";
    case Variant::const_lift: return "const-lift";
    case Variant::no_lift: return "no-lift";
  }
  return "?";
}

struct MatchParams {  // iris.hpp:157-174
  double match_ratio = 0.375;
  unsigned m = 16;
  std::uint32_t a = 1u << 14;
  std::uint32_t b = 1u << 16;
  static MatchParams make(double ratio, unsigned m_bits = 16) {
    if (!(ratio >= 0.0 && ratio <= 0.5)) throw BoundsError("match_ratio must lie in [0, 0.5]");
    MatchParams p;
    p.match_ratio = ratio;
    p.m = m_bits;
    p.b = 1u << m_bits;
    const double x = (1.0 - 2.0 * ratio) * p.b;
    p.a = static_cast<std::uint32_t>(x + 0.5);
    if (p.a > p.b) p.a = p.b;
    return p;
  }
};

struct EngineConfig {  // engine.hpp:33-44
  Backend backend = Backend::shamir;
  Variant variant = Variant::mpc_lift;
  std::uint32_t l = 12800;
  MatchParams params{};
  unsigned rotations = 31;
  bool debug_rows = false;
};

struct QueryStats {
  std::string variant = "mpc-lift", backend;
  std::uint64_t s = 0, l = 0, batch = 0;
  std::uint64_t dot_bytes = 0, lift_bytes = 0, msb_bytes = 0, or_tree_bytes = 0;
  std::uint64_t dot_rounds = 0, lift_rounds = 0, msb_rounds = 0, or_tree_rounds = 0;
  double wall_ms = 0.0;
};

struct MembershipResult {
  std::vector<std::uint8_t> person_match;  // filled for P1
  std::vector<std::uint8_t> row_bits;      // debug mode, P1
  QueryStats stats;
  std::uint64_t lane_count = 0;
};

using Payloads = std::array<std::span<const std::uint8_t>, 3>;

inline std::array<std::uint8_t, 48> seeds_from_master(std::uint64_t seed) {
  std::array<std::uint8_t, 48> s{};
  irismpc_gpu_seeds_from_master(seed, s.data());
  return s;
}

// All three parties of one DB shard on one B200.
class Session {
 public:
  Session(const EngineConfig& cfg, const std::array<std::uint8_t, 48>& seeds, int device = 0,
          std::uint32_t shard_rank = 0, std::uint64_t db_rows_total = 0, std::uint64_t db_row_offset = 0)
      : cfg_(cfg) {
    irismpc_gpu_config c{};
    c.backend = static_cast<std::uint32_t>(cfg.backend);
    c.variant = static_cast<std::uint32_t>(cfg.variant);
    c.match_ratio = cfg.params.match_ratio;
    c.l = cfg.l;
    c.a = cfg.params.a;
    c.b = cfg.params.b;
    c.m = cfg.params.m;
    c.rotations = cfg.rotations;
    c.debug_rows = cfg.debug_rows ? 1 : 0;
    for (int i = 0; i < 48; ++i) c.seeds[i] = seeds[i];
    c.device = device;
    c.shard_rank = shard_rank;
    c.db_rows_total = db_rows_total;
    c.db_row_offset = db_row_offset;
    check(irismpc_gpu_create(&c, &ctx_), "irismpc_gpu_create");
  }
  ~Session() { irismpc_gpu_destroy(ctx_); }
  Session(const Session&) = delete;
  Session& operator=(const Session&) = delete;

  void load_db(const Payloads& payload, std::uint64_t s) {  // Session::load_db
    const std::uint8_t* p[3] = {payload[0].data(), payload[1].data(), payload[2].data()};
    const std::size_t len[3] = {payload[0].size(), payload[1].size(), payload[2].size()};
    check(irismpc_gpu_load_db(ctx_, p, len, s), "load_db", ctx_);
    s_ = s;
  }

  std::array<MembershipResult, 3> batch_query(const Payloads& q, unsigned persons) {
    return query(q, persons, false);
  }
  std::array<MembershipResult, 3> membership(const Payloads& q) { return query(q, 1, true); }

  // Streaming (irismpc_gpu_batch_query_submit / _wait): DEVICE payloads that stay valid
  // until the ticket completes; at most two queries in flight on the device (a third
  // submit first completes the oldest, whose bits are kept here).  wait() returns P1's bits.
  std::uint64_t submit(const std::array<const std::uint8_t*, 3>& dq, const std::array<std::size_t, 3>& qlen,
                       unsigned persons) {
    std::size_t inflight = 0;
    for (const auto& e : pending_) inflight += !e.done;
    if (inflight >= 2)
      for (auto& e : pending_)
        if (!e.done) {
          complete(e);
          break;
        }
    Pending e{0, std::make_unique<std::vector<std::uint8_t>>(persons, 0), false};  // stable while in flight
    check(irismpc_gpu_batch_query_submit(ctx_, dq.data(), qlen.data(), persons, e.bits->data(), &e.ticket),
          "submit", ctx_);
    pending_.push_back(std::move(e));
    return pending_.back().ticket;
  }
  std::vector<std::uint8_t> wait(std::uint64_t ticket) {
    for (auto it = pending_.begin(); it != pending_.end(); ++it)
      if (it->ticket == ticket) {
        if (!it->done) complete(*it);
        std::vector<std::uint8_t> r = std::move(*it->bits);
        pending_.erase(it);
        return r;
      }
    throw Error("wait: unknown ticket");
  }

  irismpc_gpu_ctx* raw() { return ctx_; }
  std::uint64_t rows() const { return s_; }

 private:
  std::array<MembershipResult, 3> query(const Payloads& q, unsigned persons, bool membership) {
    const std::uint8_t* p[3] = {q[0].data(), q[1].data(), q[2].data()};
    const std::size_t len[3] = {q[0].size(), q[1].size(), q[2].size()};
    const std::uint64_t n = irismpc_gpu_lane_count(persons, s_, membership ? 1 : cfg_.rotations, membership);
    std::array<MembershipResult, 3> out;
    auto& o = out[0];
    o.person_match.resize(persons);
    if (cfg_.debug_rows) o.row_bits.resize(n);
    irismpc_gpu_stats st{};
    const int rc = membership
                       ? irismpc_gpu_membership(ctx_, p, len, o.person_match.data(),
                                                cfg_.debug_rows ? o.row_bits.data() : nullptr, &st)
                       : irismpc_gpu_batch_query(ctx_, p, len, persons, o.person_match.data(),
                                                 cfg_.debug_rows ? o.row_bits.data() : nullptr, &st);
    check(rc, membership ? "membership" : "batch_query", ctx_);
    for (int i = 0; i < 3; ++i) {
      auto& r = out[i];
      r.lane_count = n;
      r.stats.backend = cfg_.backend == Backend::shamir ? "shamir-galois" : "replicated";
      r.stats.variant = to_string(cfg_.variant);
      r.stats.s = st.s;
      r.stats.l = st.l;
      r.stats.batch = st.batch;
      r.stats.dot_bytes = st.dot_bytes[i];
      r.stats.lift_bytes = st.lift_bytes[i];
      r.stats.msb_bytes = st.msb_bytes[i];
      r.stats.or_tree_bytes = st.or_tree_bytes[i];
      r.stats.dot_rounds = st.dot_rounds;
      r.stats.lift_rounds = st.lift_rounds;
      r.stats.msb_rounds = st.msb_rounds;
      r.stats.or_tree_rounds = st.or_tree_rounds;
      r.stats.wall_ms = st.wall_ms;
    }
    return out;
  }

  EngineConfig cfg_;
  irismpc_gpu_ctx* ctx_ = nullptr;
  std::uint64_t s_ = 0;
  struct Pending {
    std::uint64_t ticket;
    std::unique_ptr<std::vector<std::uint8_t>> bits;
    bool done;
  };
  void complete(Pending& e) {
    irismpc_gpu_stats st{};
    check(irismpc_gpu_batch_query_wait(ctx_, e.ticket, &st), "wait", ctx_);
    e.done = true;
  }
  std::vector<Pending> pending_;
};

// ---- DB-sharded queries: one Session per shard (GPU), each with
// a contiguous row range of the DB; the library broadcasts the query from
// shard 0, gathers the per-person XOR-shared partials and opens on shard 0.
class ShardGroup {  // in-process collectives (contexts of one process, one thread each)
 public:
  explicit ShardGroup(std::uint32_t world) { check(irismpc_gpu_shard_group_create(world, &h_), "shard_group"); }
  ~ShardGroup() { irismpc_gpu_shard_group_destroy(h_); }
  ShardGroup(const ShardGroup&) = delete;
  ShardGroup& operator=(const ShardGroup&) = delete;
  irismpc_gpu_shard_group* handle() const { return h_; }

 private:
  irismpc_gpu_shard_group* h_ = nullptr;
};

class ShardedSession {
 public:
  ShardedSession(const EngineConfig& cfg, const std::array<std::uint8_t, 48>& seeds, std::uint32_t rank,
                 std::uint64_t db_rows_total, std::uint64_t db_row_offset, int device = 0)
      : cfg_(cfg), rank_(rank), session_(cfg, seeds, device, rank, db_rows_total, db_row_offset) {}

  void attach(ShardGroup& g) { check(irismpc_gpu_shard_attach_inproc(session_.raw(), g.handle()), "attach", session_.raw()); }
  void attach_nccl(const std::array<std::uint8_t, 128>& id, std::uint32_t world) {
    check(irismpc_gpu_shard_attach_nccl(session_.raw(), id.data(), world), "attach_nccl", session_.raw());
  }
  // this shard's rows of the three parties' IRS1 payloads
  void load_db(const Payloads& payload, std::uint64_t rows) { session_.load_db(payload, rows); }

  // every shard calls it together; q is read on shard 0 only (others may pass
  // empty spans of the right size in qlen); person_match is filled on shard 0
  MembershipResult batch_query(const Payloads& q, unsigned persons) {
    const std::uint8_t* p[3] = {q[0].data(), q[1].data(), q[2].data()};
    const std::size_t len[3] = {q[0].size(), q[1].size(), q[2].size()};
    MembershipResult r;
    r.person_match.resize(persons);
    irismpc_gpu_stats st{};
    check(irismpc_gpu_sharded_batch_query(session_.raw(), rank_ == 0 ? p : nullptr, len, persons,
                                          r.person_match.data(), &st),
          "sharded_batch_query", session_.raw());
    if (rank_ != 0) r.person_match.clear();
    r.lane_count = st.lanes;
    r.stats.s = st.s;
    r.stats.l = st.l;
    r.stats.batch = st.batch;
    r.stats.wall_ms = st.wall_ms;
    return r;
  }
  std::uint32_t rank() const { return rank_; }
  Session& session() { return session_; }

 private:
  EngineConfig cfg_;
  std::uint32_t rank_;
  Session session_;
};

// Drop-in for the per-party entry points: three party threads rendezvous and
// the last arrival runs the fused 3-party query.  Like the reference
// (party_batch_query / party_membership load the DB on every call,
// engine.cpp:404-420), every call reloads the DB from the payloads it is given.
// A caller that keeps the DB unchanged between calls can opt into residency
// with keep_db_resident(true); it must then call invalidate_db() after
// rewriting the payload bytes in place.  Freshness is never inferred from
// pointer identity alone.
class ThreePartyGpu {
 public:
  ThreePartyGpu(const EngineConfig& cfg, std::uint64_t seed, int device = 0)
      : session_(cfg, seeds_from_master(seed), device) {}

  void keep_db_resident(bool on) {
    std::lock_guard<std::mutex> lk(mu_);
    resident_ = on;
    valid_ = false;
  }
  void invalidate_db() {
    std::lock_guard<std::mutex> lk(mu_);
    valid_ = false;
  }

  MembershipResult party_batch_query(unsigned party /* 1..3 */, std::span<const std::uint8_t> db_payload,
                                     std::uint64_t s, std::span<const std::uint8_t> query_payload, unsigned persons) {
    return arrive(party, db_payload, s, query_payload, persons, false);
  }
  MembershipResult party_membership(unsigned party, std::span<const std::uint8_t> db_payload, std::uint64_t s,
                                    std::span<const std::uint8_t> query_payload) {
    return arrive(party, db_payload, s, query_payload, 1, true);
  }

 private:
  MembershipResult arrive(unsigned party, std::span<const std::uint8_t> db, std::uint64_t s,
                          std::span<const std::uint8_t> q, unsigned persons, bool membership) {
    if (party < 1 || party > 3) throw Error("party must be 1..3");
    std::unique_lock<std::mutex> lk(mu_);
    const std::uint64_t gen = gen_;
    db_[party - 1] = db;
    q_[party - 1] = q;
    if (++arrived_ == 3) {
      arrived_ = 0;
      try {
        if (!resident_ || !valid_ || !same(db_, loaded_) || s != session_.rows()) {
          valid_ = false;
          session_.load_db(db_, s);
          loaded_ = db_;
          valid_ = true;
        }
        results_ = membership ? session_.membership(q_) : session_.batch_query(q_, persons);
        error_.clear();
      } catch (const std::exception& e) {
        error_ = e.what();
      }
      ++gen_;
      cv_.notify_all();
    } else {
      cv_.wait(lk, [&] { return gen_ != gen; });
    }
    if (!error_.empty()) throw Error(error_);
    return results_[party - 1];
  }

  static bool same(const Payloads& a, const Payloads& b) {
    for (int i = 0; i < 3; ++i)
      if (a[i].data() != b[i].data() || a[i].size() != b[i].size()) return false;
    return true;
  }

  Session session_;
  std::mutex mu_;
  std::condition_variable cv_;
  unsigned arrived_ = 0;
  std::uint64_t gen_ = 0;
  bool resident_ = false, valid_ = false;
  Payloads db_{}, q_{}, loaded_{};
  std::array<MembershipResult, 3> results_{};
  std::string error_;
};

// ---- party mode: one party per process or thread, every
// message of the protocol through a transport, like PartyCtx on a TcpMesh.
using Seed16 = std::array<std::uint8_t, 16>;

inline std::array<std::uint8_t, 128> nccl_unique_id() {
  std::array<std::uint8_t, 128> id{};
  check(irismpc_gpu_nccl_unique_id(id.data()), "nccl_unique_id");
  return id;
}

// InProcNet (transport.hpp:129-154): mailboxes for three parties in one process.
class InProcNet {
 public:
  InProcNet() { check(irismpc_gpu_inproc_create(&h_), "inproc_create"); }
  ~InProcNet() { irismpc_gpu_inproc_destroy(h_); }
  InProcNet(const InProcNet&) = delete;
  InProcNet& operator=(const InProcNet&) = delete;
  irismpc_gpu_inproc* handle() const { return h_; }

 private:
  irismpc_gpu_inproc* h_ = nullptr;
};

// One party: its own payloads and its (own, prev) seeds (read_seed_file).
class GpuParty {
 public:
  // NCCL: rank = party - 1 of a 3-rank communicator built from `nccl_id`.
  GpuParty(const EngineConfig& cfg, unsigned party, const Seed16& own, const Seed16& prev,
           const std::array<std::uint8_t, 128>& nccl_id, int device = 0)
      : cfg_(cfg), party_(party) {
    const irismpc_gpu_config c = make(cfg, own, prev, device);
    check(irismpc_gpu_party_create_nccl(&c, party, nccl_id.data(), &h_), "party_create_nccl");
  }
  // in-process: the three parties share `net`, one host thread each.
  GpuParty(const EngineConfig& cfg, unsigned party, const Seed16& own, const Seed16& prev, InProcNet& net,
           int device = 0)
      : cfg_(cfg), party_(party) {
    const irismpc_gpu_config c = make(cfg, own, prev, device);
    check(irismpc_gpu_party_create_inproc(&c, party, net.handle(), &h_), "party_create_inproc");
  }
  ~GpuParty() { irismpc_gpu_party_destroy(h_); }
  GpuParty(const GpuParty&) = delete;
  GpuParty& operator=(const GpuParty&) = delete;

  unsigned party() const { return party_; }
  std::uint64_t rows() const { return s_; }

  void load_db(std::span<const std::uint8_t> payload, std::uint64_t s) {  // Session::load_db
    pcheck(irismpc_gpu_party_load_db(h_, payload.data(), payload.size(), s), "load_db");
    s_ = s;
    loaded_ = payload;
  }
  bool loaded(std::span<const std::uint8_t> payload, std::uint64_t s) const {
    return payload.data() == loaded_.data() && payload.size() == loaded_.size() && s == s_;
  }

  // Session::batch_query / membership at this party: person_match and row_bits at P1;
  // stats = the measured ledger of this party's messages.
  MembershipResult batch_query(std::span<const std::uint8_t> q, unsigned persons) {
    return run(q, persons, false);
  }
  MembershipResult membership(std::span<const std::uint8_t> q) { return run(q, 1, true); }

 private:
  static irismpc_gpu_config make(const EngineConfig& cfg, const Seed16& own, const Seed16& prev, int device) {
    irismpc_gpu_config c{};
    c.backend = static_cast<std::uint32_t>(cfg.backend);
    c.variant = static_cast<std::uint32_t>(cfg.variant);
    c.l = cfg.l;
    c.a = cfg.params.a;
    c.b = cfg.params.b;
    c.m = cfg.params.m;
    c.match_ratio = cfg.params.match_ratio;
    c.rotations = cfg.rotations;
    c.debug_rows = cfg.debug_rows ? 1 : 0;
    for (int i = 0; i < 16; ++i) {
      c.seeds[i] = own[i];
      c.seeds[16 + i] = prev[i];
    }
    c.device = device;
    return c;
  }
  void pcheck(int rc, const char* what) {
    if (rc == IRISMPC_GPU_OK) return;
    const std::string msg = std::string(what) + ": " + irismpc_gpu_party_last_error(h_);
    switch (rc) {
      case IRISMPC_GPU_ERR_BOUNDS: throw BoundsError(msg);
      case IRISMPC_GPU_ERR_DEVICE: throw TransportError(msg);
      case IRISMPC_GPU_ERR_INCONSISTENT: throw InconsistentShareError(msg);
      default: throw Error(msg);
    }
  }
  MembershipResult run(std::span<const std::uint8_t> q, unsigned persons, bool membership) {
    MembershipResult r;
    const std::uint64_t n = irismpc_gpu_lane_count(persons, s_, membership ? 1 : cfg_.rotations, membership ? 1 : 0);
    std::vector<std::uint8_t> pm(membership ? 1 : persons), rows(cfg_.debug_rows ? n : 0);
    irismpc_gpu_party_stats st{};
    const int rc = membership
                       ? irismpc_gpu_party_membership(h_, q.data(), q.size(), pm.data(),
                                                      cfg_.debug_rows ? rows.data() : nullptr, &st)
                       : irismpc_gpu_party_batch_query(h_, q.data(), q.size(), persons, pm.data(),
                                                       cfg_.debug_rows ? rows.data() : nullptr, &st);
    pcheck(rc, membership ? "membership" : "batch_query");
    r.lane_count = n;
    if (party_ == 1) {
      r.person_match = std::move(pm);
      r.row_bits = std::move(rows);
    }
    r.stats.backend = cfg_.backend == Backend::shamir ? "shamir-galois" : "replicated";
    r.stats.variant = to_string(cfg_.variant);
    r.stats.s = st.s;
    r.stats.l = st.l;
    r.stats.batch = st.batch;
    r.stats.dot_bytes = st.dot_bytes;
    r.stats.lift_bytes = st.lift_bytes;
    r.stats.msb_bytes = st.msb_bytes;
    r.stats.or_tree_bytes = st.or_tree_bytes;
    r.stats.dot_rounds = st.dot_rounds;
    r.stats.lift_rounds = st.lift_rounds;
    r.stats.msb_rounds = st.msb_rounds;
    r.stats.or_tree_rounds = st.or_tree_rounds;
    r.stats.wall_ms = st.wall_ms;
    return r;
  }

  EngineConfig cfg_;
  unsigned party_;
  irismpc_gpu_party* h_ = nullptr;
  std::uint64_t s_ = 0;
  std::span<const std::uint8_t> loaded_{};
};

// party_batch_query(PartyCtx&, cfg, db_payload, s, query_payload, persons)
// (engine.hpp:311-313) at one party: loads the DB on every call, as the
// reference does (engine.cpp:404-420).  Callers that keep a DB resident call
// GpuParty::load_db once and GpuParty::batch_query per query instead.
inline MembershipResult party_batch_query(GpuParty& ctx, std::span<const std::uint8_t> db_payload, std::uint64_t s,
                                          std::span<const std::uint8_t> query_payload, unsigned persons) {
  ctx.load_db(db_payload, s);
  return ctx.batch_query(query_payload, persons);
}
inline MembershipResult party_membership(GpuParty& ctx, std::span<const std::uint8_t> db_payload, std::uint64_t s,
                                         std::span<const std::uint8_t> query_payload) {
  ctx.load_db(db_payload, s);
  return ctx.membership(query_payload);
}

}  // namespace irismpc_b200
