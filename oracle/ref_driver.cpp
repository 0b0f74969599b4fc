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

#include <bit>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <vector>

#include "irismpc/cluster.hpp"
#include "irismpc/engine.hpp"
#include "irismpc/galois.hpp"
#include "irismpc/io.hpp"
#include "irismpc/kernels.hpp"
#include "irismpc/prf.hpp"
#include "irismpc/shares.hpp"
#include "oracle.hpp"  // the reference's plaintext test oracle (proj/tests/oracle.hpp)

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

EngineConfig make_cfg(int backend, int variant, std::uint32_t l, double ratio, std::uint32_t rotations,
                      int debug_rows, int parallel_dot) {
  EngineConfig cfg;
  cfg.backend = backend ? Backend::shamir : Backend::replicated;
  cfg.variant = static_cast<Variant>(variant);
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

namespace {

// Rotated query instances, rotated[c][j] at offset (j - half) * l/64
// (Session::batch_query, engine.cpp:240-256).
template <typename Inst, typename Parse>
std::vector<std::vector<Inst>> rotated_queries(Parse parse, std::uint32_t ncodes, unsigned r,
                                               std::ptrdiff_t stride) {
  const int half = static_cast<int>(r - 1) / 2;
  std::vector<std::vector<Inst>> out(ncodes);
  for (std::uint32_t c = 0; c < ncodes; ++c) {
    const Inst base = parse(c);
    for (unsigned j = 0; j < r; ++j) out[c].push_back(base.rotated((static_cast<int>(j) - half) * stride));
  }
  return out;
}

// Per-party additive dots of one record field (code at byte offset 0 or the
// mask at `off`) at width K: db blocks via kernels::dot_*_rows, then the pair
// lanes via detail::*_pair_dot, in the schedule order of engine.cpp:262-293.
template <unsigned K>
void field_dots(Backend be, PartyId self, std::uint32_t l, const std::uint8_t* db, std::size_t rec,
                std::size_t off, std::uint64_t s, const std::uint8_t* q, std::uint32_t ncodes, unsigned r,
                std::uint32_t persons, bool membership, std::vector<Ring<K>>& out) {
  const std::ptrdiff_t stride = static_cast<std::ptrdiff_t>(l / 64);
  const unsigned half = (r - 1) / 2;
  const std::uint64_t ncols = static_cast<std::uint64_t>(ncodes) * r;
  if (be == Backend::replicated) {
    kernels::PrepMatrix<K> m;
    m.rows = s;
    m.len = l;
    for (std::uint64_t row = 0; row < s; ++row) {
      const std::uint8_t* p = db + row * rec + off;
      auto ci = detail::parse_rep_inst<K>(p, l);
      m.own_sum.insert(m.own_sum.end(), ci.sum.begin(), ci.sum.end());
      m.prev.insert(m.prev.end(), ci.prev.begin(), ci.prev.end());
    }
    auto qs = rotated_queries<detail::RepInst<K>>(
        [&](std::uint32_t c) {
          const std::uint8_t* p = q + c * rec + off;
          return detail::parse_rep_inst<K>(p, l);
        },
        ncodes, r, stride);
    for (std::uint64_t col = 0; col < ncols; ++col) {
      const auto& y = qs[col / r][col % r];
      kernels::dot_prep_rows<K>(m, y.sum, y.prev, std::span<Ring<K>>(out.data() + col * s, s), true);
    }
    std::uint64_t k = ncols * s;
    for (std::uint32_t i = 0; i < persons && !membership; ++i)
      for (std::uint32_t j = i + 1; j < persons; ++j)
        for (unsigned ea = 0; ea < 2; ++ea)
          for (unsigned eb = 0; eb < 2; ++eb)
            for (unsigned rot = 0; rot < r; ++rot, ++k)
              out[k] = detail::rep_pair_dot<K>(qs[2 * i + ea][rot], qs[2 * j + eb][half]);
  } else {
    kernels::GrMatrix<K> m;
    m.rows = s;
    m.len = l / 2;
    for (std::uint64_t row = 0; row < s; ++row) {
      const std::uint8_t* p = db + row * rec + off;
      auto ci = detail::parse_gr_inst<K>(p, l, self);
      m.c0.insert(m.c0.end(), ci.lc0.begin(), ci.lc0.end());
      m.c1.insert(m.c1.end(), ci.lc1.begin(), ci.lc1.end());
    }
    auto qs = rotated_queries<detail::GrInst<K>>(
        [&](std::uint32_t c) {
          const std::uint8_t* p = q + c * rec + off;
          return detail::parse_gr_inst<K>(p, l, self);
        },
        ncodes, r, stride);
    for (std::uint64_t col = 0; col < ncols; ++col) {
      const auto& y = qs[col / r][col % r];
      kernels::dot_gr_ct_rows<K>(m, y.c0, y.c1, std::span<Ring<K>>(out.data() + col * s, s), true);
    }
    std::uint64_t k = ncols * s;
    for (std::uint32_t i = 0; i < persons && !membership; ++i)
      for (std::uint32_t j = i + 1; j < persons; ++j)
        for (unsigned ea = 0; ea < 2; ++ea)
          for (unsigned eb = 0; eb < 2; ++eb)
            for (unsigned rot = 0; rot < r; ++rot, ++k)
              out[k] = detail::gr_pair_dot<K>(qs[2 * i + ea][rot], qs[2 * j + eb][half]);
  }
}

// Public-mask popcounts (engine.cpp:329-334, 349-350) over parse_mask_bits +
// BitVec::rotated; popcount_and is restated (it is file-local to engine.cpp).
void plain_ml(std::uint32_t l, const std::uint8_t* db, std::size_t rec, std::size_t off, std::uint64_t s,
              const std::uint8_t* q, std::uint32_t ncodes, unsigned r, std::uint32_t persons,
              bool membership, std::int64_t* out) {
  auto pc = [](const BitVec& a, const BitVec& b) {
    std::int64_t c = 0;
    for (std::size_t i = 0; i < a.words().size(); ++i) c += std::popcount(a.words()[i] & b.words()[i]);
    return c;
  };
  const std::ptrdiff_t stride = static_cast<std::ptrdiff_t>(l / 64);
  const int half = static_cast<int>(r - 1) / 2;
  std::vector<std::vector<BitVec>> qs(ncodes);
  for (std::uint32_t c = 0; c < ncodes; ++c) {
    const std::uint8_t* p = q + c * rec + off;
    const BitVec m = detail::parse_mask_bits(p, l);
    for (unsigned j = 0; j < r; ++j) qs[c].push_back(m.rotated((static_cast<int>(j) - half) * stride));
  }
  const std::uint64_t ncols = static_cast<std::uint64_t>(ncodes) * r;
  for (std::uint64_t row = 0; row < s; ++row) {
    const std::uint8_t* p = db + row * rec + off;
    const BitVec m = detail::parse_mask_bits(p, l);
    for (std::uint64_t col = 0; col < ncols; ++col) out[col * s + row] = pc(qs[col / r][col % r], m);
  }
  std::uint64_t k = ncols * s;
  for (std::uint32_t i = 0; i < persons && !membership; ++i)
    for (std::uint32_t j = i + 1; j < persons; ++j)
      for (unsigned ea = 0; ea < 2; ++ea)
        for (unsigned eb = 0; eb < 2; ++eb)
          for (unsigned rot = 0; rot < r; ++rot, ++k) out[k] = pc(qs[2 * i + ea][rot], qs[2 * j + eb][half]);
}

template <unsigned KH, unsigned KM>
void dots_reshare_t(Backend be, Variant v, std::uint32_t l, unsigned r, const std::array<Seed, 3>& seeds,
                    const std::uint8_t* const* db, std::uint64_t s, const std::uint8_t* const* q,
                    std::uint32_t persons, bool membership, std::uint64_t n, std::uint32_t* dot_hd,
                    std::uint32_t* dot_ml, std::int64_t* public_ml, std::uint32_t* rs_hd,
                    std::uint32_t* rs_ml) {
  const std::size_t crec = code_record_bytes(be, v, l);
  const std::size_t rec = crec + mask_record_bytes(be, v, l);
  const std::uint32_t ncodes = membership ? 1 : 2 * persons;
  if (KM == 0 && public_ml) plain_ml(l, db[0], rec, crec, s, q[0], ncodes, r, persons, membership, public_ml);
  for (unsigned pi = 0; pi < 3; ++pi) {
    const PartyId self = static_cast<PartyId>(pi + 1);
    std::vector<Ring<KH>> hd(n);
    field_dots<KH>(be, self, l, db[pi], rec, 0, s, q[pi], ncodes, r, persons, membership, hd);
    constexpr unsigned KMs = KM == 0 ? 16 : KM;
    std::vector<Ring<KMs>> ml(KM == 0 ? 0 : n);
    if constexpr (KM != 0)
      field_dots<KM>(be, self, l, db[pi], rec, crec, s, q[pi], ncodes, r, persons, membership, ml);
    // reshare_pair<KH, KM> order (engine.cpp:80-106): hd lanes, then ml lanes.
    SeedPair sp = seed_pair_for(self, seeds);
    for (std::uint64_t i = 0; i < n; ++i) {
      if (dot_hd) dot_hd[pi * n + i] = static_cast<std::uint32_t>(hd[i].value());
      const auto z = hd[i] + sp.zero_ring<KH>();
      if (rs_hd) rs_hd[pi * n + i] = static_cast<std::uint32_t>(z.value());
    }
    for (std::uint64_t i = 0; i < ml.size(); ++i) {
      if (dot_ml) dot_ml[pi * n + i] = static_cast<std::uint32_t>(ml[i].value());
      const auto z = ml[i] + sp.zero_ring<KMs>();
      if (rs_ml) rs_ml[pi * n + i] = static_cast<std::uint32_t>(z.value());
    }
  }
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
std::uint64_t ref_deal(int backend, int variant, std::uint32_t l, std::uint64_t seed, std::uint64_t tag,
                       std::uint64_t nrec, const std::uint64_t* codes, const std::uint64_t* masks,
                       std::uint8_t* out1, std::uint8_t* out2, std::uint8_t* out3) {
  IrisDb db(l);
  const std::size_t wl = (l + 63) / 64;
  for (std::uint64_t r = 0; r < nrec; ++r) db.add(to_record(l, codes + r * wl, masks + r * wl));
  Rng rng(CtrPrf::derive(CtrPrf::seed_from_u64(seed), tag));
  const auto pay = deal_db_payload(db, backend ? Backend::shamir : Backend::replicated,
                                   static_cast<Variant>(variant), rng);
  std::memcpy(out1, pay[0].data(), pay[0].size());
  std::memcpy(out2, pay[1].data(), pay[1].size());
  std::memcpy(out3, pay[2].data(), pay[2].size());
  return pay[0].size();
}

// run_batch_local / run_membership_local.  stats: [3][8] per party
// (dot, lift, msb, or bytes; dot, lift, msb, or rounds); wall_ms: max over
// parties of QueryStats.wall_ms (run_schedule only).
int ref_run_local(int backend, int variant, std::uint32_t l, double ratio, std::uint32_t rotations,
                  int debug_rows, int parallel_dot, std::uint64_t seed, std::uint64_t s,
                  const std::uint64_t* db_codes, const std::uint64_t* db_masks,
                  std::uint32_t persons, const std::uint64_t* q_codes,
                  const std::uint64_t* q_masks, int membership, std::uint8_t* person_match,
                  std::uint8_t* row_bits, std::uint64_t* stats, double* wall_ms,
                  std::uint64_t* lanes) {
  try {
    const auto cfg = make_cfg(backend, variant, l, ratio, rotations, debug_rows, parallel_dot);
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


// L1 + L2: per-party additive dot outputs (mod 2^KH / 2^KM; public popcounts
// for plain-mask) and reshared components, computed with the reference's
// parse/dot kernels and SeedPair zero shares in the reshare_pair order.
// Arrays are [party][lane].
int ref_dots_reshare(int backend, int variant, std::uint32_t l, std::uint32_t rotations,
                     const std::uint8_t seeds48[48], const std::uint8_t* const* db,
                     std::uint64_t s, const std::uint8_t* const* q, std::uint32_t persons,
                     int membership, std::uint32_t* dot_hd, std::uint32_t* dot_ml,
                     std::int64_t* public_ml, std::uint32_t* rs_hd, std::uint32_t* rs_ml) {
  try {
    const Backend be = backend ? Backend::shamir : Backend::replicated;
    const Variant v = static_cast<Variant>(variant);
    const unsigned r = membership ? 1 : rotations;
    const std::uint32_t ncodes = membership ? 1 : 2 * persons;
    const std::uint64_t n = static_cast<std::uint64_t>(ncodes) * r * s +
        (membership ? 0 : static_cast<std::uint64_t>(persons) * (persons ? persons - 1 : 0) / 2 * 4 * r);
    std::array<Seed, 3> seeds;
    for (int k = 0; k < 3; ++k) std::memcpy(seeds[k].bytes.data(), seeds48 + 16 * k, 16);
    const bool m = membership != 0;
    switch (v) {
      case Variant::plain_mask:
        dots_reshare_t<16, 0>(be, v, l, r, seeds, db, s, q, persons, m, n, dot_hd, dot_ml, public_ml, rs_hd, rs_ml);
        break;
      case Variant::mpc_lift:
        dots_reshare_t<16, 16>(be, v, l, r, seeds, db, s, q, persons, m, n, dot_hd, dot_ml, public_ml, rs_hd, rs_ml);
        break;
      case Variant::const_lift:
        dots_reshare_t<16, 32>(be, v, l, r, seeds, db, s, q, persons, m, n, dot_hd, dot_ml, public_ml, rs_hd, rs_ml);
        break;
      case Variant::no_lift:
        dots_reshare_t<32, 32>(be, v, l, r, seeds, db, s, q, persons, m, n, dot_hd, dot_ml, public_ml, rs_hd, rs_ml);
        break;
      default:
        return 2;
    }
    return 0;
  } catch (...) {
    return map_error();
  }
}

// --- files (io.cpp) ---------------------------------------------------------

// write_iris_db of the given records (io.cpp:74-88)
int ref_write_iris_db(const char* path, std::uint32_t l, std::uint64_t s, const std::uint64_t* codes,
                      const std::uint64_t* masks) {
  try {
    IrisDb db(l);
    const std::size_t wl = (l + 63) / 64;
    for (std::uint64_t r = 0; r < s; ++r) db.add(to_record(l, codes + r * wl, masks + r * wl));
    write_iris_db(path, db);
    return 0;
  } catch (...) {
    return map_error();
  }
}

// The `irismpc share` dealer (tools/irismpc_cli.cpp:137-172) for one variant:
// read_iris_db, seeds deal_seeds(Rng(derive(seed_from_u64(seed), 0x5eed))),
// payload deal_db_payload with Rng(derive(seed_from_u64(seed), variant + 1)),
// one IRSD + one IRS1 file per party.  (The CLI itself needs CLI11, which is
// not vendored; this calls the same library functions in the same order.)
int ref_share_files(const char* db_path, int backend, int variant, std::uint64_t seed,
                    const char* const* share_paths, const char* const* seed_paths) {
  try {
    const auto db = read_iris_db(db_path);
    const Backend be = backend ? Backend::shamir : Backend::replicated;
    const Variant v = static_cast<Variant>(variant);
    Rng seed_rng(CtrPrf::derive(CtrPrf::seed_from_u64(seed), 0x5eed));
    const auto seeds = deal_seeds(seed_rng);
    for (unsigned p = 1; p <= 3; ++p) {
      const auto prev = seeds[party_index(prev_party(static_cast<PartyId>(p))) - 1];
      write_seed_file(seed_paths[p - 1], p, seeds[p - 1], prev);
    }
    Rng rng(CtrPrf::derive(CtrPrf::seed_from_u64(seed), static_cast<std::uint64_t>(v) + 1));
    const auto payload = deal_db_payload(db, be, v, rng);
    for (unsigned p = 1; p <= 3; ++p) {
      ShareFileHeader h;
      h.backend = be;
      h.variant = v;
      h.party = p;
      h.l = db.l;
      h.s = db.size();
      write_share_file(share_paths[p - 1], h, payload[p - 1]);
    }
    return 0;
  } catch (...) {
    return map_error();
  }
}

// read_share_file: header fields + payload size (2 on the reference's errors)
int ref_read_share_file(const char* path, std::uint32_t* hdr, std::uint64_t* s, std::uint64_t* payload_len) {
  try {
    const auto [h, bytes] = read_share_file(path);
    hdr[0] = static_cast<std::uint32_t>(h.backend);
    hdr[1] = static_cast<std::uint32_t>(h.variant);
    hdr[2] = h.party;
    hdr[3] = h.l;
    *s = h.s;
    *payload_len = bytes.size();
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
void* ref_bench_prepare(int backend, int variant, std::uint32_t l, std::uint64_t s, std::uint32_t persons) {
  auto* b = new RefBench;
  b->cfg = make_cfg(backend, variant, l, 0.375, 31, 0, 1);
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

// or_tree_batch (circuits.hpp:387-434) run by the reference over caller-given
// bit sharings: comps [3][total] component bits (party p's own = component
// p - 1, its prev = the previous party's), groups = consecutive runs of lens[g]
// lanes; the parties' seeds from run_parties(seed), streams at 0.  Writes the
// aggregate's components [3][ngroups] (each party's own share of lane g).
int ref_or_tree_batch_shares(std::uint32_t ngroups, const std::uint64_t* lens, const std::uint8_t* comps,
                             std::uint64_t total, std::uint64_t seed, std::uint8_t* agg) {
  try {
    auto results = run_parties(seed, [&](PartyCtx& ctx) {
      const unsigned own = party_index(ctx.id) - 1, prv = party_index(prev_party(ctx.id)) - 1;
      std::vector<OrTreeInput> groups;
      std::uint64_t off = 0;
      for (std::uint32_t g = 0; g < ngroups; ++g) {
        OrTreeInput in{BitRow(lens[g]), lens[g]};
        for (std::uint64_t i = 0; i < lens[g]; ++i)
          in.bits.set_lane(i, BitWord{comps[own * total + off + i], comps[prv * total + off + i]});
        off += lens[g];
        groups.push_back(std::move(in));
      }
      auto [out, st] = or_tree_batch(ctx, std::move(groups));
      (void)st;
      std::vector<std::uint8_t> mine(ngroups);
      for (std::uint32_t g = 0; g < ngroups; ++g) mine[g] = (std::uint8_t)(out.lane(g).own & 1);
      return mine;
    });
    for (int p = 0; p < 3; ++p)
      for (std::uint32_t g = 0; g < ngroups; ++g) agg[p * ngroups + g] = std::get<0>(results[p])[g];
    return 0;
  } catch (...) {
    return map_error();
  }
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


// --- the reference's randomized equivalence grid (tests/equiv_common.hpp) ---

namespace {
void put_record(const IrisRecord& r, std::uint64_t* c, std::uint64_t* m) {
  for (std::size_t i = 0; i < r.code.words().size(); ++i) {
    c[i] = r.code.words()[i];
    m[i] = r.mask.words()[i];
  }
}
EngineConfig grid_config(int backend, int variant, std::uint32_t l, double ratio) {
  EngineConfig cfg;
  cfg.backend = backend ? Backend::shamir : Backend::replicated;
  cfg.variant = static_cast<Variant>(variant);
  cfg.l = l;
  cfg.params = MatchParams::make(ratio, 16);
  cfg.debug_rows = true;
  return cfg;
}
}  // namespace

// One run_instance of equiv_common.hpp:61-89, generated with the reference's
// own Rng / random_record in the same draw order (DB rows with a mask density
// drawn from {0, 1, 0.3, 0.85}, a random query, one time in three a noisy
// planted copy of a row), then run through run_membership_local (debug rows)
// and the plaintext oracle::naive_membership.  Outputs the instance records,
// want (oracle), got (reference aggregate) and the reference's row bits.
int ref_equiv_instance(int backend, int variant, std::uint32_t l, std::uint64_t s, std::uint64_t seed, double ratio,
                       std::uint64_t* db_codes, std::uint64_t* db_masks, std::uint64_t* q_code,
                       std::uint64_t* q_mask, std::uint8_t* want, std::uint8_t* got, std::uint8_t* row_bits) {
  try {
    const std::size_t wl = (l + 63) / 64;
    Rng rng(seed * 2654435761u + l * 97 + s);
    IrisDb db(l);
    for (std::uint64_t i = 0; i < s; ++i) {
      const std::uint64_t pick = rng.below(5);
      const double density = pick == 0 ? 0.0 : pick == 1 ? 1.0 : pick == 2 ? 0.3 : 0.85;
      db.add(random_record(l, rng, density));
    }
    IrisRecord q = random_record(l, rng, 0.85);
    if (s > 0 && rng.below(3) == 0) {
      q = db.rows[rng.below(s)];
      for (int f = 0; f < 4; ++f) {
        const std::size_t i = rng.below(l);
        q.code.set(i, !q.code.get(i));
      }
    }
    const auto cfg = grid_config(backend, variant, l, ratio);
    const auto out = run_membership_local(cfg, q, db, seed);
    *want = oracle::naive_membership(q, db, cfg.params, cfg.variant) ? 1 : 0;
    *got = out.aggregate() ? 1 : 0;
    for (std::uint64_t i = 0; i < s; ++i) {
      put_record(db.rows[i], db_codes + i * wl, db_masks + i * wl);
      row_bits[i] = out.output().row_bits.at(i);
    }
    put_record(q, q_code, q_mask);
    return 0;
  } catch (...) {
    return map_error();
  }
}

// run_boundary_instances (equiv_common.hpp:93-128): `count` full-mask l = 64
// pairs with b*dot at a*ml and one dot step either side, for ratios 0.375 and
// 0.3, cycling backend (made % 2) and variant ((made / 2) % 4).  Per instance:
// backend, variant, ratio, the membership seed, the row, the query, want, got.
int ref_boundary_instances(unsigned count, int* backend, int* variant, double* ratio, std::uint64_t* mseed,
                           std::uint64_t* row_code, std::uint64_t* row_mask, std::uint64_t* q_code,
                           std::uint64_t* q_mask, std::uint8_t* want, std::uint8_t* got) {
  try {
    const std::size_t l = 64;
    std::uint64_t seed = 0xb0;
    const double ratios[2] = {0.375, 0.3};
    unsigned made = 0;
    while (made < count) {
      for (const double rt : ratios) {
        const auto params = MatchParams::make(rt, 16);
        const double target = static_cast<double>(params.a) * l / params.b;
        for (int delta = -1; delta <= 1 && made < count; ++delta) {
          const std::int64_t hd = (static_cast<std::int64_t>(l) - static_cast<std::int64_t>(target)) / 2 + delta;
          if (hd < 0 || hd > static_cast<std::int64_t>(l)) continue;
          Rng rng(seed++);
          IrisRecord row(BitVec::random(l, rng), BitVec(l));
          for (std::size_t i = 0; i < l; ++i) row.mask.set(i, true);
          IrisRecord q = row;
          for (std::int64_t i = 0; i < hd; ++i)
            q.code.set(static_cast<std::size_t>(i), !q.code.get(static_cast<std::size_t>(i)));
          IrisDb db(l);
          db.add(row);
          backend[made] = static_cast<int>(made % 2 == 0 ? 0 : 1);  // backends[2] = {replicated, shamir}
          variant[made] = static_cast<int>((made / 2) % 4);
          ratio[made] = rt;
          mseed[made] = seed;
          const auto cfg = grid_config(backend[made], variant[made], static_cast<std::uint32_t>(l), rt);
          const auto out = run_membership_local(cfg, q, db, seed);
          want[made] = oracle::naive_membership(q, db, cfg.params, cfg.variant) ? 1 : 0;
          got[made] = out.aggregate() ? 1 : 0;
          put_record(row, row_code + made, row_mask + made);
          put_record(q, q_code + made, q_mask + made);
          ++made;
        }
      }
    }
    return 0;
  } catch (...) {
    return map_error();
  }
}

// test_engine.cpp:42-82: planted self-match (7 random rows + a full-mask query
// row), its complement, and the ml = 0 instance; k = 0, 1, 2 selects which.
// Records out (up to 8 rows), want/got as above.
int ref_engine_case(int which, int backend, int variant, std::uint64_t* db_codes, std::uint64_t* db_masks,
                    std::uint64_t* s_out, std::uint64_t* q_code, std::uint64_t* q_mask, std::uint8_t* want,
                    std::uint8_t* got) {
  try {
    const std::size_t l = 64;
    IrisDb db(l);
    IrisRecord q{BitVec(l), BitVec(l)};
    std::uint64_t mseed = 500;
    if (which == 0 || which == 1) {
      Rng rng(101);
      for (int i = 0; i < 7; ++i) db.add(random_record(l, rng, 0.8));
      q = IrisRecord(BitVec::random(l, rng), BitVec(l));
      for (std::size_t i = 0; i < l; ++i) q.mask.set(i, true);
      db.add(q);
      if (which == 1) {
        IrisRecord comp = q;
        for (std::size_t i = 0; i < l; ++i) comp.code.set(i, !q.code.get(i));
        db = IrisDb(l);
        db.add(comp);
        mseed = 501;
      }
    } else {
      Rng rng(102);
      q = IrisRecord(BitVec::random(l, rng), BitVec(l));
      IrisRecord row(q.code, BitVec(l));
      for (std::size_t i = 0; i < 32; ++i) q.mask.set(i, true);
      for (std::size_t i = 32; i < 64; ++i) row.mask.set(i, true);
      db.add(row);
      mseed = 502;
    }
    const auto cfg = grid_config(backend, variant, static_cast<std::uint32_t>(l), 0.375);
    const auto out = run_membership_local(cfg, q, db, mseed);
    *want = oracle::naive_membership(q, db, cfg.params, cfg.variant) ? 1 : 0;
    *got = out.aggregate() ? 1 : 0;
    *s_out = db.size();
    for (std::size_t i = 0; i < db.size(); ++i) put_record(db.rows[i], db_codes + i, db_masks + i);
    put_record(q, q_code, q_mask);
    return 0;
  } catch (...) {
    return map_error();
  }
}

// --- the comparison phase alone (the reference's `bench --phase comparison`) ---

// run_comparison_local (cluster.cpp:97-145) on plaintext (masked dot, ml)
// lanes: opened aggregate (with_or), per-party ledger bytes of the lift, ot,
// msb and or_tree phases ([3][4]) and the slowest party's wall ms.
int ref_comparison_local(int variant, std::uint64_t n, const std::int64_t* dots, const std::int64_t* mls,
                         int with_or, std::uint64_t seed, std::uint8_t* opened, std::uint64_t* ledger,
                         double* wall_ms) {
  try {
    EngineConfig cfg;
    cfg.backend = Backend::replicated;
    cfg.variant = static_cast<Variant>(variant);
    cfg.l = 12800;
    cfg.params = MatchParams::make(0.375, 16);
    std::vector<std::pair<std::int64_t, std::int64_t>> lanes(n);
    for (std::uint64_t i = 0; i < n; ++i) lanes[i] = {dots[i], mls[i]};
    const auto out = run_comparison_local(cfg, lanes, with_or != 0, seed);
    for (int p = 0; p < 3; ++p) {
      ledger[4 * p + 0] = out.ledgers[p].phase(Phase::lift).bytes_sent;
      ledger[4 * p + 1] = out.ledgers[p].phase(Phase::ot).bytes_sent;
      ledger[4 * p + 2] = out.ledgers[p].phase(Phase::msb).bytes_sent;
      ledger[4 * p + 3] = out.ledgers[p].phase(Phase::or_tree).bytes_sent;
    }
    if (opened) *opened = out.party[0].opened.empty() ? 0 : out.party[0].opened[0];
    if (wall_ms) *wall_ms = out.wall_ms;
    return 0;
  } catch (...) {
    return map_error();
  }
}

// run_or_tree_local (cluster.cpp:147-186): opened OR, or_tree bytes per party, wall ms
int ref_or_tree_local(std::uint64_t n, const std::uint8_t* bits, std::uint64_t seed, std::uint8_t* opened,
                      std::uint64_t* or_bytes, double* wall_ms) {
  try {
    const auto out = run_or_tree_local(std::span<const std::uint8_t>(bits, n), seed);
    for (int p = 0; p < 3; ++p) or_bytes[p] = out.ledgers[p].phase(Phase::or_tree).bytes_sent;
    *opened = out.aggregate ? 1 : 0;
    if (wall_ms) *wall_ms = out.wall_ms;
    return 0;
  } catch (...) {
    return map_error();
  }
}

}  // extern "C"
