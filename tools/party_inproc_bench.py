#!/usr/bin/env python3
"""Party mode with the three parties in one process on one GPU (in-process
mailbox), configs[1]-shaped; for per-kernel profiling of the party kernels
(`ncu ... python tools/party_inproc_bench.py`).  Prints one JSON line."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_2405_04463_b200 as P
    rows = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
    persons, l, r, seed = 16, 12800, 31, 7
    be = P.SHAMIR
    dealer = P.Session(P.EngineConfig(backend=be, l=l, rotations=1), master_seed=seed)
    wl = l // 64
    codes = torch.empty((rows, wl), dtype=torch.int64, device="cuda")
    masks = torch.empty((rows, wl), dtype=torch.int64, device="cuda")
    dealer.synth_records(2, 0, rows, 0.9, codes, masks)
    pay = [torch.empty(rows * dealer.rec, dtype=torch.uint8, device="cuda") for _ in range(3)]
    dealer.deal_payload(seed, 1, 0, codes, masks, pay)
    qc = torch.empty((2 * persons, wl), dtype=torch.int64, device="cuda")
    qm = torch.empty((2 * persons, wl), dtype=torch.int64, device="cuda")
    dealer.synth_records(2, rows, 2 * persons, 0.9, qc, qm)
    qc[0], qm[0] = codes[rows // 2], masks[rows // 2]
    qp = [torch.empty(2 * persons * dealer.rec, dtype=torch.uint8, device="cuda") for _ in range(3)]
    dealer.deal_payload(seed, 2, 0, qc, qm, qp)
    db = [x.cpu().numpy() for x in pay]
    q = [x.cpu().numpy() for x in qp]
    del dealer, pay, qp, codes, masks
    torch.cuda.empty_cache()
    cfg = P.EngineConfig(backend=be, l=l, rotations=r)
    t0 = time.perf_counter()
    parties = P.run_parties_inproc(cfg, P.seeds_from_master(seed), db, rows, q, persons)
    dt = time.perf_counter() - t0
    st = parties[0].last_stats
    print(json.dumps({"rows": rows, "person_match0": int(parties[0].result[0]), "host_s_incl_load": dt,
                      "p1_device_ms": st.wall_ms, "phase_ms": list(st.phase_ms)}))


if __name__ == "__main__":
    main()
