// C++ drop-in check: three party threads call ThreePartyGpu::party_batch_query
// (the reference's per-party entry point shape, engine.hpp:311-313) and P1's
// person_match must equal the oracle's; error paths map to the reference's
// exception types.  Built and run by tests/test_cpp_shim.py.
#include <algorithm>
#include <cstdio>
#include <memory>
#include <thread>
#include <vector>

#include <cuda_runtime_api.h>

#include "../../include/irismpc_b200.hpp"
#include "../../oracle/irismpc_oracle.h"

using namespace irismpc_b200;

int main() {
  const std::uint32_t l = 12800, persons = 3;
  const std::uint64_t s = 500, seed = 99;
  const int be = ORC_SHAMIR;
  const std::uint32_t wl = l / 64;
  std::vector<std::uint64_t> dc(s * wl), dm(s * wl), qc(2 * persons * wl), qm(2 * persons * wl);
  orc_rng* rng = orc_rng_new(seed);
  for (std::uint64_t r = 0; r < s; ++r) orc_rng_record(rng, l, 0.9, &dc[r * wl], &dm[r * wl]);
  for (std::uint32_t r = 0; r < 2 * persons; ++r) orc_rng_record(rng, l, 0.9, &qc[r * wl], &qm[r * wl]);
  orc_rng_free(rng);
  for (std::uint32_t w = 0; w < wl; ++w) {  // person 1's right eye is DB row 123
    qc[3 * wl + w] = dc[123 * wl + w];
    qm[3 * wl + w] = dm[123 * wl + w];
  }
  const std::size_t rec = orc_code_record_bytes(be, ORC_MPC_LIFT, l) + orc_mask_record_bytes(be, ORC_MPC_LIFT, l);
  std::array<std::vector<std::uint8_t>, 3> db, q;
  for (int p = 0; p < 3; ++p) {
    db[p].resize(s * rec);
    q[p].resize(2 * persons * rec);
  }
  orc_rng* dr = orc_rng_sub(seed, 1);
  orc_rng* qr = orc_rng_sub(seed, 2);
  orc_deal_payload(be, l, s, dc.data(), dm.data(), dr, db[0].data(), db[1].data(), db[2].data());
  orc_deal_payload(be, l, 2 * persons, qc.data(), qm.data(), qr, q[0].data(), q[1].data(), q[2].data());
  orc_rng_free(dr);
  orc_rng_free(qr);

  orc_config oc{be, ORC_MPC_LIFT, l, orc_match_a(0.375), 1u << 16, 31, 0, 0.375};
  std::vector<std::uint8_t> want(persons);
  orc_out out{};
  out.person_match = want.data();
  std::uint8_t seeds[48];
  orc_party_seeds(seed, seeds);
  if (orc_query(&oc, seeds, db[0].data(), db[1].data(), db[2].data(), s, q[0].data(), q[1].data(),
                q[2].data(), persons, 0, nullptr, &out) != 0) {
    std::puts("oracle failed");
    return 2;
  }

  EngineConfig cfg;
  cfg.backend = Backend::shamir;
  cfg.l = l;
  cfg.params = MatchParams::make(0.375, 16);
  cfg.rotations = 31;
  ThreePartyGpu gpu(cfg, seed);
  for (int round = 0; round < 2; ++round) {  // reloads the DB every call, like the reference
    std::array<MembershipResult, 3> res;
    std::vector<std::thread> th;
    for (unsigned p = 1; p <= 3; ++p)
      th.emplace_back([&, p] { res[p - 1] = gpu.party_batch_query(p, db[p - 1], s, q[p - 1], persons); });
    for (auto& t : th) t.join();
    if (round == 0 && res[0].person_match != want) {
      std::printf("MISMATCH person_match\n");
      return 1;
    }
    if (res[0].lane_count != irismpc_gpu_lane_count(persons, s, 31, 0)) return 1;
    if (res[1].stats.lift_bytes != res[2].stats.lift_bytes) return 1;  // P2, P3 send 4n OT bytes
  }
  if (want[1] != 1) return 1;

  // in-place rewrite of the DB payload bytes between calls (same buffers, same
  // sizes): row 123 becomes a copy of row 0's shares, so person 1's planted match
  // must disappear -- the shim reloads the DB every call (engine.cpp:404-420)
  {
    const auto orig = db;
    for (int p = 0; p < 3; ++p) std::copy(orig[p].begin(), orig[p].begin() + rec, db[p].begin() + 123 * rec);
    std::vector<std::uint8_t> want3(persons);
    orc_out o3{};
    o3.person_match = want3.data();
    if (orc_query(&oc, seeds, db[0].data(), db[1].data(), db[2].data(), s, q[0].data(), q[1].data(), q[2].data(),
                  persons, 0, nullptr, &o3) != 0)
      return 2;
    std::array<MembershipResult, 3> res;
    std::vector<std::thread> th;
    for (unsigned p = 1; p <= 3; ++p)
      th.emplace_back([&, p] { res[p - 1] = gpu.party_batch_query(p, db[p - 1], s, q[p - 1], persons); });
    for (auto& t : th) t.join();
    if (res[0].person_match != want3 || want3[1] != 0) {
      std::printf("MISMATCH after in-place DB rewrite\n");
      return 1;
    }
    for (int p = 0; p < 3; ++p) std::copy(orig[p].begin(), orig[p].end(), db[p].begin());
  }

  // DB-sharded query through the C-ABI: two shards of the same DB on
  // this GPU in one process, an in-process shard group, one thread per shard
  {
    const auto& dbo = db;
    const std::uint64_t split = 217;
    ShardGroup group(2);
    std::array<std::unique_ptr<ShardedSession>, 2> sh;
    for (std::uint32_t r = 0; r < 2; ++r) {
      const std::uint64_t r0 = r == 0 ? 0 : split, r1 = r == 0 ? split : s;
      sh[r] = std::make_unique<ShardedSession>(cfg, seeds_from_master(seed), r, s, r0);
      sh[r]->attach(group);
      Payloads part;
      for (int p = 0; p < 3; ++p) part[p] = std::span<const std::uint8_t>(dbo[p].data() + r0 * rec, (r1 - r0) * rec);
      sh[r]->load_db(part, r1 - r0);
    }
    std::array<MembershipResult, 2> res;
    std::vector<std::thread> th;
    for (std::uint32_t r = 0; r < 2; ++r)
      th.emplace_back([&, r] { res[r] = sh[r]->batch_query({q[0], q[1], q[2]}, persons); });
    for (auto& t : th) t.join();
    if (res[0].person_match != want) {
      std::printf("MISMATCH sharded person_match\n");
      return 1;
    }
  }

  // streaming: Session::submit / wait with device query payloads, three submits
  // (the third completes the oldest implicitly), every ticket equals the oracle
  {
    Session st(cfg, seeds_from_master(seed));
    st.load_db({db[0], db[1], db[2]}, s);
    std::array<std::uint8_t*, 3> dq{};
    std::array<std::size_t, 3> qlen{};
    for (int p = 0; p < 3; ++p) {
      qlen[p] = q[p].size();
      if (cudaMalloc(reinterpret_cast<void**>(&dq[p]), qlen[p]) != cudaSuccess ||
          cudaMemcpy(dq[p], q[p].data(), qlen[p], cudaMemcpyHostToDevice) != cudaSuccess)
        return 2;
    }
    const std::array<const std::uint8_t*, 3> cq{dq[0], dq[1], dq[2]};
    std::uint64_t t[3];
    for (int i = 0; i < 3; ++i) t[i] = st.submit(cq, qlen, persons);
    for (int i = 2; i >= 0; --i)
      if (st.wait(t[i]) != want) {
        std::printf("MISMATCH streaming ticket %d\n", i);
        return 1;
      }
    for (int p = 0; p < 3; ++p) cudaFree(dq[p]);
  }

  // party mode: three GpuParty objects on one InProcNet, one thread each,
  // the reference's per-party call shape; P1's bits and every party's
  // measured ledger equal the oracle's (the reference's QueryStats)
  {
    orc_stats ost[3];
    orc_out o2{};
    std::vector<std::uint8_t> want2(persons);
    o2.person_match = want2.data();
    o2.stats = ost;
    if (orc_query(&oc, seeds, db[0].data(), db[1].data(), db[2].data(), s, q[0].data(), q[1].data(), q[2].data(),
                  persons, 0, nullptr, &o2) != 0)
      return 2;
    InProcNet net;
    std::array<std::unique_ptr<GpuParty>, 3> pt;
    for (unsigned p = 1; p <= 3; ++p) {
      Seed16 own{}, prev{};
      const unsigned pv = (p + 1) % 3;  // index of seed_{p-1} (p = 1..3 -> 2, 0, 1)
      for (int i = 0; i < 16; ++i) {
        own[i] = seeds[16 * (p - 1) + i];
        prev[i] = seeds[16 * pv + i];
      }
      pt[p - 1] = std::make_unique<GpuParty>(cfg, p, own, prev, net);
    }
    std::array<MembershipResult, 3> res;
    std::vector<std::thread> th;
    for (unsigned p = 1; p <= 3; ++p)
      th.emplace_back([&, p] { res[p - 1] = party_batch_query(*pt[p - 1], db[p - 1], s, q[p - 1], persons); });
    for (auto& t : th) t.join();
    if (res[0].person_match != want2) {
      std::printf("MISMATCH party-mode person_match\n");
      return 1;
    }
    for (int p = 0; p < 3; ++p) {
      const auto& st = res[p].stats;
      if (st.dot_bytes != ost[p].dot_bytes || st.lift_bytes != ost[p].lift_bytes || st.msb_bytes != ost[p].msb_bytes ||
          st.or_tree_bytes != ost[p].or_tree_bytes || st.lift_rounds != ost[p].lift_rounds ||
          st.or_tree_rounds != ost[p].or_tree_rounds) {
        std::printf("MISMATCH party-mode ledger P%d\n", p + 1);
        return 1;
      }
    }
  }

  // error mapping: db payload size mismatch -> Error (engine.cpp:142)
  Session sess(cfg, seeds_from_master(seed));
  bool threw = false;
  try {
    sess.load_db({std::span<const std::uint8_t>(db[0].data(), 7), db[1], db[2]}, s);
  } catch (const Error&) {
    threw = true;
  }
  if (!threw) return 1;
  // bounds: Shamir with an odd rotation stride (engine.cpp:31-33)
  threw = false;
  try {
    EngineConfig bad = cfg;
    bad.l = 192;
    Session b(bad, seeds_from_master(seed));
  } catch (const BoundsError&) {
    threw = true;
  }
  if (!threw) return 1;
  std::printf("shim ok: person_match = %d %d %d\n", want[0], want[1], want[2]);
  return 0;
}
