// Thin extern "C" driver around the UNMODIFIED reference library
// (/root/reference/proj, compiled from its own sources by oracle/Makefile into
// oracle/_ref/libirismpc_ref.so).  TEST INFRASTRUCTURE ONLY: it lets tests/
// pin the C restatement (irismpc_oracle.c) against the reference itself and
// lets bench.py time the reference CPU path (the `--impl reference` arm).
//
// Every entry point only calls reference code: run_batch_local /
// run_membership_local (cluster.cpp:30-79), deal_*_payload (shares.cpp:76-90),
// kernels::dot_*_rows (kernels.cpp:29-53), detail::parse_*_inst and the
// SeedPair zero shares in the order of reshare_pair (engine.cpp:80-106).

#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <vector>

#include "irismpc/cluster.hpp"
#include "irismpc/engine.hpp"
#include "irismpc/galois.hpp"
#include "irismpc/kernels.hpp"
#include "irismpc/prf.hpp"
#include "irismpc/shares.hpp"

using namespace irismpc;

namespace {

IrisRecord to_record(std::uint32_t l, const std::uint64_t* code, const std::uint64_t* mask) {
  BitVec c(l), m(l);
  const std::size_t wl = (l + 63) / 64;
  for (std::size_t i = 0; i < wl; ++i) {
    c.words()[i] = code[i];
    m.words()[i] = mask[i];
  }
  return IrisRecord(std::move(c), std::move(m));
}

EngineConfig make_cfg(int backend, std::uint32_t l, double ratio, std::uint32_t rotations,
                      int debug_rows, int parallel_dot) {
  EngineConfig cfg;
  cfg.backend = backend ? Backend::shamir : Backend::replicated;
  cfg.variant = Variant::mpc_lift;
  cfg.l = l;
  cfg.params = MatchParams::make(ratio, 16);
  cfg.rotations = rotations;
  cfg.debug_rows = debug_rows != 0;
  cfg.parallel_dot = parallel_dot != 0;
  return cfg;
}

int map_error() {
  try {
    throw;
  } catch (const BoundsError&) {
    return 4;
  } catch (const InconsistentShareError&) {
    return 5;
  } catch (const TransportError&) {
    return 3;
  } catch (const Error&) {
    return 2;
  } catch (...) {
    return 1;
  }
}

void fill_stats(const MembershipResult& r, std::uint64_t* st) {
  st[0] = r.stats.dot_bytes;
  st[1] = r.stats.lift_bytes;
  st[2] = r.stats.msb_bytes;
  st[3] = r.stats.or_tree_bytes;
  st[4] = r.stats.dot_rounds;
  st[5] = r.stats.lift_rounds;
  st[6] = r.stats.msb_rounds;
  st[7] = r.stats.or_tree_rounds;
}

}  // namespace

extern "C" {

void ref_chacha_block(const std::uint8_t seed[16], std::uint64_t block, std::uint64_t stream,
                      std::uint32_t out[16]) {
  Seed s;
  std::memcpy(s.bytes.data(), seed, 16);
  detail::chacha_block(s, block, stream, out);
}

void ref_seed_from_u64(std::uint64_t v, std::uint8_t out[16]) {
  const Seed s = CtrPrf::seed_from_u64(v);
  std::memcpy(out, s.bytes.data(), 16);
}

void ref_party_seeds(std::uint64_t master, std::uint8_t out[48]) {
  Rng seed_rng(CtrPrf::derive(CtrPrf::seed_from_u64(master), 0x5eed));
  const auto seeds = deal_seeds(seed_rng);
  for (int k = 0; k < 3; ++k) std::memcpy(out + 16 * k, seeds[k].bytes.data(), 16);
}

void ref_rng_u64(std::uint64_t seed, std::uint64_t n, std::uint64_t* out) {
  Rng rng(seed);
  for (std::uint64_t i = 0; i < n; ++i) out[i] = rng.next_u64();
}

// `count` random_record(l, Rng(seed), density[i]) draws in sequence.
void ref_random_records(std::uint64_t seed, std::uint32_t l, std::uint64_t count,
                        const double* density, std::uint64_t* codes, std::uint64_t* masks) {
  Rng rng(seed);
  const std::size_t wl = (l + 63) / 64;
  for (std::uint64_t r = 0; r < count; ++r) {
    const IrisRecord rec = random_record(l, rng, density[r]);
    for (std::size_t i = 0; i < wl; ++i) {
      codes[r * wl + i] = rec.code.words()[i];
      masks[r * wl + i] = rec.mask.words()[i];
    }
  }
}

void ref_lambda16(std::uint16_t out[6]) {
  const auto lam = party_lagrange_at_zero<16>();
  for (int i = 0; i < 3; ++i) {
    out[2 * i] = lam[i].c0.value();
    out[2 * i + 1] = lam[i].c1.value();
  }
}

// deal_db_payload with sub_rng(seed, tag) (cluster.cpp:24-26,55-57).
std::uint64_t ref_deal(int backend, std::uint32_t l, std::uint64_t seed, std::uint64_t tag,
                       std::uint64_t nrec, const std::uint64_t* codes, const std::uint64_t* masks,
                       std::uint8_t* out1, std::uint8_t* out2, std::uint8_t* out3) {
  IrisDb db(l);
  const std::size_t wl = (l + 63) / 64;
  for (std::uint64_t r = 0; r < nrec; ++r) db.add(to_record(l, codes + r * wl, masks + r * wl));
  Rng rng(CtrPrf::derive(CtrPrf::seed_from_u64(seed), tag));
  const auto pay = deal_db_payload(db, backend ? Backend::shamir : Backend::replicated,
                                   Variant::mpc_lift, rng);
  std::memcpy(out1, pay[0].data(), pay[0].size());
  std::memcpy(out2, pay[1].data(), pay[1].size());
  std::memcpy(out3, pay[2].data(), pay[2].size());
  return pay[0].size();
}

// run_batch_local / run_membership_local.  stats: [3][8] per party
// (dot, lift, msb, or bytes; dot, lift, msb, or rounds); wall_ms: max over
// parties of QueryStats.wall_ms (run_schedule only).
int ref_run_local(int backend, std::uint32_t l, double ratio, std::uint32_t rotations,
                  int debug_rows, int parallel_dot, std::uint64_t seed, std::uint64_t s,
                  const std::uint64_t* db_codes, const std::uint64_t* db_masks,
                  std::uint32_t persons, const std::uint64_t* q_codes,
                  const std::uint64_t* q_masks, int membership, std::uint8_t* person_match,
                  std::uint8_t* row_bits, std::uint64_t* stats, double* wall_ms,
                  std::uint64_t* lanes) {
  try {
    const auto cfg = make_cfg(backend, l, ratio, rotations, debug_rows, parallel_dot);
    const std::size_t wl = (l + 63) / 64;
    IrisDb db(l);
    for (std::uint64_t r = 0; r < s; ++r) db.add(to_record(l, db_codes + r * wl, db_masks + r * wl));
    LocalOutcome out;
    if (membership) {
      out = run_membership_local(cfg, to_record(l, q_codes, q_masks), db, seed);
    } else {
      std::vector<std::pair<IrisRecord, IrisRecord>> batch;
      for (std::uint32_t i = 0; i < persons; ++i) {
        batch.emplace_back(to_record(l, q_codes + (2 * i) * wl, q_masks + (2 * i) * wl),
                           to_record(l, q_codes + (2 * i + 1) * wl, q_masks + (2 * i + 1) * wl));
      }
      out = run_batch_local(cfg, batch, db, seed);
    }
    const auto& o = out.output();
    if (person_match) std::memcpy(person_match, o.person_match.data(), o.person_match.size());
    if (row_bits && !o.row_bits.empty()) std::memcpy(row_bits, o.row_bits.data(), o.row_bits.size());
    double w = 0;
    for (int p = 0; p < 3; ++p) {
      if (stats) fill_stats(out.party[p], stats + 8 * p);
      w = out.party[p].stats.wall_ms > w ? out.party[p].stats.wall_ms : w;
    }
    if (wall_ms) *wall_ms = w;
    if (lanes) *lanes = o.lane_count;
    return 0;
  } catch (...) {
    return map_error();
  }
}

// L1 + L2: per-party additive dot outputs and reshared components, computed
// with the reference's parse/dot kernels and SeedPair zero shares in the
// reshare_pair order.  Arrays are [party][lane].
int ref_dots_reshare(int backend, std::uint32_t l, std::uint32_t rotations,
                     const std::uint8_t seeds48[48], const std::uint8_t* const* db,
                     std::uint64_t s, const std::uint8_t* const* q, std::uint32_t persons,
                     int membership, std::uint16_t* dot_hd, std::uint16_t* dot_ml,
                     std::uint16_t* rs_hd, std::uint16_t* rs_ml) {
  try {
    const Backend be = backend ? Backend::shamir : Backend::replicated;
    const std::size_t crec = code_record_bytes(be, Variant::mpc_lift, l);
    const std::size_t rec = crec + mask_record_bytes(be, Variant::mpc_lift, l);
    const unsigned r = membership ? 1 : rotations;
    const int half = static_cast<int>(r - 1) / 2;
    const std::ptrdiff_t stride = static_cast<std::ptrdiff_t>(l / 64);
    const std::uint32_t ncodes = membership ? 1 : 2 * persons;
    const std::uint64_t ncols = static_cast<std::uint64_t>(ncodes) * r;
    const std::uint64_t npairs =
        membership ? 0 : static_cast<std::uint64_t>(persons) * (persons ? persons - 1 : 0) / 2 * 4 * r;
    const std::uint64_t n = ncols * s + npairs;
    std::array<Seed, 3> seeds;
    for (int k = 0; k < 3; ++k) std::memcpy(seeds[k].bytes.data(), seeds48 + 16 * k, 16);

    for (unsigned pi = 0; pi < 3; ++pi) {
      const PartyId self = static_cast<PartyId>(pi + 1);
      std::vector<R16> hd(n), ml(n);
      if (be == Backend::replicated) {
        kernels::PrepMatrix<16> mc, mm;
        mc.rows = mm.rows = s;
        mc.len = mm.len = l;
        for (std::uint64_t row = 0; row < s; ++row) {
          const std::uint8_t* p = db[pi] + row * rec;
          auto ci = detail::parse_rep_inst<16>(p, l);
          auto mi = detail::parse_rep_inst<16>(p, l);
          mc.own_sum.insert(mc.own_sum.end(), ci.sum.begin(), ci.sum.end());
          mc.prev.insert(mc.prev.end(), ci.prev.begin(), ci.prev.end());
          mm.own_sum.insert(mm.own_sum.end(), mi.sum.begin(), mi.sum.end());
          mm.prev.insert(mm.prev.end(), mi.prev.begin(), mi.prev.end());
        }
        std::vector<std::vector<detail::RepInst<16>>> qc(ncodes), qm(ncodes);
        for (std::uint32_t c = 0; c < ncodes; ++c) {
          const std::uint8_t* p = q[pi] + c * rec;
          auto ci = detail::parse_rep_inst<16>(p, l);
          auto mi = detail::parse_rep_inst<16>(p, l);
          for (unsigned j = 0; j < r; ++j) {
            const std::ptrdiff_t by = (static_cast<int>(j) - half) * stride;
            qc[c].push_back(ci.rotated(by));
            qm[c].push_back(mi.rotated(by));
          }
        }
        for (std::uint64_t col = 0; col < ncols; ++col) {
          const auto& yc = qc[col / r][col % r];
          const auto& ym = qm[col / r][col % r];
          kernels::dot_prep_rows<16>(mc, yc.sum, yc.prev, std::span<R16>(hd.data() + col * s, s), true);
          kernels::dot_prep_rows<16>(mm, ym.sum, ym.prev, std::span<R16>(ml.data() + col * s, s), true);
        }
        std::uint64_t k = ncols * s;
        for (std::uint32_t i = 0; i < persons && !membership; ++i)
          for (std::uint32_t j = i + 1; j < persons; ++j)
            for (unsigned ea = 0; ea < 2; ++ea)
              for (unsigned eb = 0; eb < 2; ++eb)
                for (unsigned rot = 0; rot < r; ++rot, ++k) {
                  hd[k] = detail::rep_pair_dot<16>(qc[2 * i + ea][rot], qc[2 * j + eb][half]);
                  ml[k] = detail::rep_pair_dot<16>(qm[2 * i + ea][rot], qm[2 * j + eb][half]);
                }
      } else {
        kernels::GrMatrix<16> mc, mm;
        mc.rows = mm.rows = s;
        mc.len = mm.len = l / 2;
        for (std::uint64_t row = 0; row < s; ++row) {
          const std::uint8_t* p = db[pi] + row * rec;
          auto ci = detail::parse_gr_inst<16>(p, l, self);
          auto mi = detail::parse_gr_inst<16>(p, l, self);
          mc.c0.insert(mc.c0.end(), ci.lc0.begin(), ci.lc0.end());
          mc.c1.insert(mc.c1.end(), ci.lc1.begin(), ci.lc1.end());
          mm.c0.insert(mm.c0.end(), mi.lc0.begin(), mi.lc0.end());
          mm.c1.insert(mm.c1.end(), mi.lc1.begin(), mi.lc1.end());
        }
        std::vector<std::vector<detail::GrInst<16>>> qc(ncodes), qm(ncodes);
        for (std::uint32_t c = 0; c < ncodes; ++c) {
          const std::uint8_t* p = q[pi] + c * rec;
          auto ci = detail::parse_gr_inst<16>(p, l, self);
          auto mi = detail::parse_gr_inst<16>(p, l, self);
          for (unsigned j = 0; j < r; ++j) {
            const std::ptrdiff_t by = (static_cast<int>(j) - half) * stride;
            qc[c].push_back(ci.rotated(by));
            qm[c].push_back(mi.rotated(by));
          }
        }
        for (std::uint64_t col = 0; col < ncols; ++col) {
          const auto& yc = qc[col / r][col % r];
          const auto& ym = qm[col / r][col % r];
          kernels::dot_gr_ct_rows<16>(mc, yc.c0, yc.c1, std::span<R16>(hd.data() + col * s, s), true);
          kernels::dot_gr_ct_rows<16>(mm, ym.c0, ym.c1, std::span<R16>(ml.data() + col * s, s), true);
        }
        std::uint64_t k = ncols * s;
        for (std::uint32_t i = 0; i < persons && !membership; ++i)
          for (std::uint32_t j = i + 1; j < persons; ++j)
            for (unsigned ea = 0; ea < 2; ++ea)
              for (unsigned eb = 0; eb < 2; ++eb)
                for (unsigned rot = 0; rot < r; ++rot, ++k) {
                  hd[k] = detail::gr_pair_dot<16>(qc[2 * i + ea][rot], qc[2 * j + eb][half]);
                  ml[k] = detail::gr_pair_dot<16>(qm[2 * i + ea][rot], qm[2 * j + eb][half]);
                }
      }
      // reshare_pair<16,16> order: hd lanes then ml lanes, own = z + zero_ring.
      SeedPair sp = seed_pair_for(self, seeds);
      for (std::uint64_t i = 0; i < n; ++i) {
        if (dot_hd) dot_hd[pi * n + i] = hd[i].value();
        if (rs_hd) rs_hd[pi * n + i] = (hd[i] + sp.zero_ring<16>()).value();
      }
      for (std::uint64_t i = 0; i < n; ++i) {
        if (dot_ml) dot_ml[pi * n + i] = ml[i].value();
        if (rs_ml) rs_ml[pi * n + i] = (ml[i] + sp.zero_ring<16>()).value();
      }
      if (!rs_hd && !rs_ml) continue;
    }
    return 0;
  } catch (...) {
    return map_error();
  }
}

// --- reference CPU timing (the bench.py `--impl reference` arm) ----------

struct RefBench {
  EngineConfig cfg;
  std::array<std::vector<std::uint8_t>, 3> db, q;
  std::uint64_t s;
  unsigned persons;
};

// Deals a synthetic workload: DB rows random_record(l, Rng(2), 0.9),
// then 2*persons query codes from the same stream; person 0's left eye is a planted
// copy of row s/2.  Dealing seed 7: DB sub_rng(7,1), queries sub_rng(7,2).
void* ref_bench_prepare(int backend, std::uint32_t l, std::uint64_t s, std::uint32_t persons) {
  auto* b = new RefBench;
  b->cfg = make_cfg(backend, l, 0.375, 31, 0, 1);
  b->s = s;
  b->persons = persons;
  Rng rng(2);
  IrisDb db(l);
  for (std::uint64_t i = 0; i < s; ++i) db.add(random_record(l, rng, 0.9));
  std::vector<IrisRecord> codes;
  for (std::uint32_t i = 0; i < 2 * persons; ++i) codes.push_back(random_record(l, rng, 0.9));
  if (s > 0 && persons > 0) {
    // planted near-match: row s/2 rotated by +2 strides, 4 code bits flipped
    const IrisRecord& src = db.rows[s / 2];
    const std::ptrdiff_t by = 2 * static_cast<std::ptrdiff_t>(l / 64);
    IrisRecord p(src.code.rotated(by), src.mask.rotated(by));
    for (std::uint32_t f = 0; f < 4; ++f) {
      const std::size_t i = f * (l / 4) + 7;
      p.code.set(i, !p.code.get(i));
    }
    codes[0] = p;
  }
  Rng drng(CtrPrf::derive(CtrPrf::seed_from_u64(7), 1));
  Rng qrng(CtrPrf::derive(CtrPrf::seed_from_u64(7), 2));
  b->db = deal_db_payload(db, b->cfg.backend, b->cfg.variant, drng);
  b->q = deal_query_payload(codes, b->cfg.backend, b->cfg.variant, qrng);
  return b;
}

// One step: the three parties run party_batch_query (stock path).  Returns
// the slowest party's QueryStats.wall_ms; person 0's opened bit in *match0.
double ref_bench_step(void* h, std::uint8_t* match0) {
  auto* b = static_cast<RefBench*>(h);
  auto results = run_parties(7, [&](PartyCtx& ctx) {
    const unsigned i = party_index(ctx.id) - 1;
    return party_batch_query(ctx, b->cfg, b->db[i], b->s, b->q[i], b->persons);
  });
  double w = 0;
  for (int p = 0; p < 3; ++p) {
    const auto& r = std::get<0>(results[p]);
    w = r.stats.wall_ms > w ? r.stats.wall_ms : w;
  }
  if (match0) *match0 = std::get<0>(results[0]).person_match.at(0);
  return w;
}

void ref_bench_free(void* h) { delete static_cast<RefBench*>(h); }

}  // extern "C"
