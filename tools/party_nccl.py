#!/usr/bin/env python3
"""Party mode over NCCL: three ranks = parties 1, 2, 3, one GPU each.

    torchrun --nproc-per-node 3 --master-addr 127.0.0.1 tools/party_nccl.py --check      # parity vs the oracle
    torchrun --nproc-per-node 3 --master-addr 127.0.0.1 tools/party_nccl.py --rows 100000  # timing, configs[1]

Each rank holds only its own party's payloads and seeds (dealt on the device,
bit-identical to the reference dealer) and exchanges every protocol message
with the other two over NCCL send/recv.  Rank 0 (= P1) prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=100_000)
    ap.add_argument("--persons", type=int, default=16)
    ap.add_argument("--l", type=int, default=12800)
    ap.add_argument("--rotations", type=int, default=31)
    ap.add_argument("--backend", default="shamir", choices=["shamir", "replicated"])
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--variant", default="mpc-lift", choices=["plain-mask", "mpc-lift", "const-lift", "no-lift"])
    ap.add_argument("--check", action="store_true", help="small case, every share vs the oracle")
    a = ap.parse_args()

    import torch
    import torch.distributed as dist
    import paper_2405_04463_b200 as P

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    assert world == 3, "party mode runs exactly three ranks (parties 1, 2, 3)"
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")  # plumbing only: the ncclUniqueId broadcast
    idt = torch.zeros(128, dtype=torch.uint8)
    if rank == 0:
        idt.copy_(torch.frombuffer(bytearray(P.nccl_unique_id()), dtype=torch.uint8))
    dist.broadcast(idt, 0)
    nccl_id = bytes(idt.numpy())

    be = P.SHAMIR if a.backend == "shamir" else P.REPLICATED
    seed = 7
    if a.check:
        a.rows, a.persons, a.l, a.rotations = 300, 3, 256, 5
    var = P.VARIANTS[a.variant]
    cfg = P.EngineConfig(backend=be, l=a.l, rotations=a.rotations, debug_rows=a.check, variant=var)
    seeds = P.seeds_from_master(seed)
    party = P.Party(cfg, rank + 1, P.party_seeds(seeds, rank + 1), nccl_id=nccl_id, device=local)

    # deal on the device (every rank deals all three payloads and keeps its own)
    dealer = P.Session(P.EngineConfig(backend=be, l=a.l, rotations=1, variant=var), master_seed=seed, device=local)
    wl = (a.l + 63) // 64
    s, ncodes = a.rows, 2 * a.persons
    codes = torch.empty((s, wl), dtype=torch.int64, device="cuda")
    masks = torch.empty((s, wl), dtype=torch.int64, device="cuda")
    dealer.synth_records(2, 0, s, 0.9, codes, masks)
    pay = [torch.empty(s * dealer.rec, dtype=torch.uint8, device="cuda") for _ in range(3)]
    dealer.deal_payload(seed, 1, 0, codes, masks, pay)
    qc = torch.empty((ncodes, wl), dtype=torch.int64, device="cuda")
    qm = torch.empty((ncodes, wl), dtype=torch.int64, device="cuda")
    dealer.synth_records(2, s, ncodes, 0.9, qc, qm)
    qc[0], qm[0] = codes[s // 2], masks[s // 2]  # person 0's left eye is DB row s/2
    qp = [torch.empty(ncodes * dealer.rec, dtype=torch.uint8, device="cuda") for _ in range(3)]
    dealer.deal_payload(seed, 2, 0, qc, qm, qp)
    my_db = pay[rank].cpu().numpy()
    my_q = qp[rank].cpu().numpy()
    all_db = [x.cpu().numpy() for x in pay] if (a.check and rank == 0) else None
    all_q = [x.cpu().numpy() for x in qp] if (a.check and rank == 0) else None
    del dealer, pay, qp, codes, masks
    torch.cuda.empty_cache()

    party.load_db(my_db, s)
    for _ in range(a.warmup if not a.check else 0):
        party.batch_query(my_q, a.persons)
    dist.barrier()
    ms = []
    out = None
    for _ in range(max(1, a.steps if not a.check else 1)):
        dist.barrier()
        t0 = time.perf_counter()
        out = party.batch_query(my_q, a.persons, want_rows=a.check)
        ms.append((time.perf_counter() - t0) * 1e3)
    st = party.last_stats
    led = torch.tensor(list(st.ledger().values()), dtype=torch.int64)
    leds = [torch.zeros_like(led) for _ in range(3)]
    dist.all_gather(leds, led)
    wall = torch.tensor([float(np.median(ms)), st.wall_ms] + list(st.phase_ms)[:6], dtype=torch.float64)
    walls = [torch.zeros_like(wall) for _ in range(3)]
    dist.all_gather(walls, wall)
    line = None
    if rank == 0:
        n = P.lane_count(a.persons, s, a.rotations)
        keys = list(st.ledger().keys())
        ledgers = [dict(zip(keys, [int(v) for v in x.tolist()])) for x in leds]
        host_ms = max(w[0].item() for w in walls)
        cmp_ = ncodes * a.rotations * s
        line = {"mode": "party (3 ranks over NCCL, one GPU per party)", "backend": a.backend, "variant": a.variant,
                "rows": s,
                "persons": a.persons, "lanes": n, "person_match": [int(x) for x in out],
                "ms_per_query_max_over_parties": host_ms,
                "device_ms": [round(w[1].item(), 3) for w in walls],
                "phase_ms_p1": dict(zip(["gemm", "dot_reshare", "lift_inject", "msb", "or_open", "in_transport"],
                                        [round(x, 3) for x in walls[0][2:].tolist()])),
                "comparisons_per_s": cmp_ / (host_ms / 1e3), "ledgers": ledgers,
                "wire_bytes_p1": int(st.wire_bytes)}
        if a.check:
            from oracle import pyoracle as O
            ref = O.query(O.make_config(be, a.l, 0.375, a.rotations, debug_rows=True, variant=var), seeds, all_db, s,
                          all_q, a.persons, want_all=True)
            line["check"] = {
                "person_match": bool((out == ref.person_match).all()),
                "row_bits": bool((party.row_bits[:n] == ref.row_bits).all()),
                "ledgers": all(ledgers[i] == ref.stats[i] for i in range(3)),
            }
        print(json.dumps(line), flush=True)
    dist.barrier()
    party.close()
    dist.destroy_process_group()
    if a.check and rank == 0 and not all(line["check"].values()):
        return 1
    return 0


if __name__ == "__main__":
    sys.exit(main())
