"""`irismpc` command line on the B200 path (reference tools/irismpc_cli.cpp).

    python -m paper_2405_04463_b200.cli gen-db --size 1000 --length 12800 --seed 1 --out db.irmp
    python -m paper_2405_04463_b200.cli share --db db.irmp --backend shamir-galois --variant all --out-dir shares
    python -m paper_2405_04463_b200.cli query --shares shares --query q.irmp --batch 16 --variant all --stats st.json
    python -m paper_2405_04463_b200.cli bench --phase full --db-size 100000 --variant mpc-lift --json b.json
    python -m paper_2405_04463_b200.cli bench [--phase comparison] --comparisons 100000 --variant all

Same subcommands, options, file names (db.<variant>.p<k>.irs, seeds.p<k>.irsd),
dealer seeds/tags, stdout lines, stats JSON (stats_to_json, irismpc_cli.cpp:103-119)
and exit codes (2 config, 3 device/transport, 4 bounds) as the reference.  The
three parties run in this process on one GPU, so `party` (the TCP party loop)
does not exist here, and `query` takes the share directory (`--shares`, or
`--config` with the reference's JSON whose `share_dir`, `backend`, `l`,
`match_ratio`, `rotations` are honoured; `endpoints` is ignored).  All compute
(record generation, dealing, queries) runs on the GPU.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

import paper_2405_04463_b200 as P

BACKENDS = {"replicated": P.REPLICATED, "shamir-galois": P.SHAMIR, "shamir": P.SHAMIR}
BACKEND_NAMES = {P.REPLICATED: "replicated", P.SHAMIR: "shamir-galois"}
VARIANT_NAMES = {v: k for k, v in P.VARIANTS.items()}


def share_path(d, v, p):  # irismpc_cli.cpp:93-97
    return os.path.join(d, f"db.{VARIANT_NAMES[v]}.p{p}.irs")


def seed_path(d, p):  # irismpc_cli.cpp:99-101
    return os.path.join(d, f"seeds.p{p}.irsd")


def stats_to_json(st: P.Stats, variant: int, backend: int, party: int = 0) -> dict:
    """stats_to_json (irismpc_cli.cpp:103-119) for one party (P1 = 0)."""
    return {"variant": VARIANT_NAMES[variant], "backend": BACKEND_NAMES[backend], "s": st.s, "l": st.l,
            "batch": st.batch,
            "phase_bytes": {"dot": st.dot_bytes[party], "lift": st.lift_bytes[party], "msb": st.msb_bytes[party],
                            "or_tree": st.or_tree_bytes[party]},
            "rounds": {"dot": st.dot_rounds, "lift": st.lift_rounds, "msb": st.msb_rounds,
                       "or_tree": st.or_tree_rounds},
            "wall_ms": st.wall_ms}


def _variants(name: str, query: bool = False):
    if name == "all":
        # the query command's "all" skips plain-mask (irismpc_cli.cpp:286-288)
        return [P.MPC_LIFT, P.CONST_LIFT, P.NO_LIFT] if query else [P.PLAIN_MASK, P.MPC_LIFT, P.CONST_LIFT,
                                                                    P.NO_LIFT]
    if name not in P.VARIANTS:
        raise P.ConfigError(f"unknown variant: {name}")
    return [P.VARIANTS[name]]


def _device_records(sess: P.Session, rng_seed: int, first: int, count: int, density: float):
    import torch
    wl = (sess.cfg.l + 63) // 64
    codes = torch.empty((max(1, count), wl), dtype=torch.int64, device="cuda")
    masks = torch.empty((max(1, count), wl), dtype=torch.int64, device="cuda")
    if count:
        sess.synth_records(rng_seed, first, count, density, codes, masks)
    return codes[:count], masks[:count]


def cmd_gen_db(a) -> int:
    """random_record(l, Rng(seed), density) x size -> IRMP (irismpc_cli.cpp:122-133)."""
    sess = P.Session(P.EngineConfig(backend=P.SHAMIR, l=a.length, rotations=1), master_seed=0)
    codes, masks = _device_records(sess, a.seed, 0, a.size, a.mask_density)
    P.write_iris_db(a.out, codes.cpu().numpy().view(np.uint64), masks.cpu().numpy().view(np.uint64), a.length)
    print(f"wrote {a.out}: s={a.size} l={a.length} ({os.path.getsize(a.out)} bytes)")
    return 0


def cmd_share(a) -> int:
    """The dealer (irismpc_cli.cpp:137-172): seeds from derive(seed, 0x5eed), payload of
    variant v from Rng(derive(seed_from_u64(seed), v + 1)), dealt on the GPU in row chunks."""
    import torch
    codes, masks, l = P.read_iris_db(a.db)
    backend = BACKENDS[a.backend]
    os.makedirs(a.out_dir, exist_ok=True)
    seeds = P.seeds_from_master(a.seed)
    for p in range(3):
        q = (p + 2) % 3
        P.write_seed_file(seed_path(a.out_dir, p + 1), p + 1, seeds[16 * p:16 * p + 16], seeds[16 * q:16 * q + 16])
    s = codes.shape[0]
    for v in _variants(a.variant):
        sess = P.Session(P.EngineConfig(backend=backend, l=l, rotations=1, variant=v), seeds=seeds)
        paths = [share_path(a.out_dir, v, p + 1) for p in range(3)]
        for p in range(3):
            P.write_share_file(paths[p], backend, v, p + 1, l, s, b"")
        chunk = max(1, (256 << 20) // max(1, sess.rec))
        for r0 in range(0, s, chunk):
            nr = min(chunk, s - r0)
            dc = torch.from_numpy(np.ascontiguousarray(codes[r0:r0 + nr]).view(np.int64)).cuda()
            dm = torch.from_numpy(np.ascontiguousarray(masks[r0:r0 + nr]).view(np.int64)).cuda()
            outs = [torch.empty(nr * sess.rec, dtype=torch.uint8, device="cuda") for _ in range(3)]
            sess.deal_payload(a.seed, v + 1, r0, dc, dm, outs)
            for p in range(3):
                with open(paths[p], "ab") as f:
                    f.write(outs[p].cpu().numpy().tobytes())
        for path in paths:
            print(f"wrote {path} ({os.path.getsize(path)} bytes)")
    return 0


def _load_query_cfg(a):
    cfg = {"share_dir": a.shares, "backend": a.backend, "l": a.length, "match_ratio": a.match_ratio,
           "rotations": a.rotations}
    if a.config:
        with open(a.config) as f:
            j = json.load(f)
        for k in cfg:
            if k in j and (k != "share_dir" or not a.shares):
                cfg[k] = j[k]
    if not cfg["share_dir"]:
        raise P.ConfigError("query needs --shares or --config with share_dir")
    return cfg


def cmd_query(a) -> int:
    """cmd_query (irismpc_cli.cpp:280-330): the query codes are dealt per variant with
    Rng(derive(seed_from_u64(seed), 0x9e + v)); the parties' PRF streams persist
    across the variants of one session, as in the party loop's PartyCtx."""
    import torch
    cfg = _load_query_cfg(a)
    backend = BACKENDS[cfg["backend"]]
    qc, qm, ql = P.read_iris_db(a.query)
    if ql != cfg["l"]:
        raise P.ConfigError("query length does not match config")
    if a.batch > 0 and qc.shape[0] != 2 * a.batch:
        raise P.ConfigError("batch query file must hold 2 codes per person")
    if a.batch == 0 and qc.shape[0] != 1:
        raise P.ConfigError("membership query file must hold 1 record")
    seeds = P.read_seed_files([seed_path(cfg["share_dir"], p) for p in (1, 2, 3)])
    pos = np.zeros(3, np.uint64)
    replies, stats = [], []
    for v in _variants(a.variant, query=True):
        rot = cfg["rotations"] if a.batch > 0 else 1
        ecfg = P.EngineConfig(backend=backend, l=cfg["l"], match_ratio=cfg["match_ratio"], rotations=rot, variant=v)
        sess = P.Session(ecfg, seeds=seeds)
        sess.load_db_files([share_path(cfg["share_dir"], v, p) for p in (1, 2, 3)])
        sess.set_stream_positions(pos)
        dc = torch.from_numpy(np.ascontiguousarray(qc).view(np.int64)).cuda()
        dm = torch.from_numpy(np.ascontiguousarray(qm).view(np.int64)).cuda()
        q = [torch.empty(qc.shape[0] * sess.rec, dtype=torch.uint8, device="cuda") for _ in range(3)]
        sess.deal_payload(a.seed, 0x9E + v, 0, dc, dm, q)
        if a.batch > 0:
            m = [bool(x) for x in sess.batch_query(q, a.batch)]
        else:
            m = [sess.membership(q)]
        pos = sess.stream_positions()
        replies.append(m)
        stats.append(stats_to_json(sess.last_stats, v, backend))
        print(f"variant {VARIANT_NAMES[v]}:" + "".join(" true" if x else " false" for x in m))
        sess.close()
    if any(r != replies[0] for r in replies[1:]):
        raise P.IrisError("variants disagree on the match outcome")
    if len(replies) > 1:
        print("all variants agree")
    if a.stats:
        with open(a.stats, "w") as f:
            json.dump(stats[0] if len(stats) == 1 else stats, f, indent=2)
            f.write("\n")
        print(f"stats written to {a.stats}")
    return 0


# PAPER.md:477-485 (Table 3): comparison phase, 100k parallel comparisons, Ryzen 9
# 7950X, one thread per party: ms, M elements/s, kB per party
PAPER_TABLE3 = {"plain-mask": (3.18, 31.4, 362), "mpc-lift": (14.47, 6.9, 2138), "const-lift": (5.32, 18.8, 763),
                "no-lift": (5.27, 19.0, 763), "or-tree": (0.87, 114.9, 12)}


def cmd_bench_comparison(a) -> int:
    """bench --phase comparison (cmd_bench, irismpc_cli.cpp:373-458; the CLI's
    default): each variant's comparison phase alone (party_comparison_only) over
    replicated shares of synthetic (masked dot, ml) lanes -- ml uniform in
    [0, l], hd uniform in [0, ml], dot = ml - 2 hd -- then the OR-tree row
    (party_or_tree_only over `comparisons` bits with one planted 1).  Best of
    --repeat device times of the comparison kernels (the payload upload over PCIe
    and its parse are reported separately as upload_parse_ms); kB/party = (lift + ot + msb bytes) averaged over the
    parties, or_tree bytes without the final 1-bit open, as the reference prints.
    The lane values come from numpy rather than the reference's Rng(1) (no
    column depends on them)."""
    n = a.comparisons
    variants = [P.PLAIN_MASK, P.MPC_LIFT, P.CONST_LIFT, P.NO_LIFT] if a.variant == "all" else [P.VARIANTS[a.variant]]
    rng = np.random.default_rng(1)
    ml = rng.integers(0, a.length + 1, n)
    hd = (rng.random(n) * (ml + 1)).astype(np.int64)
    dot = ml - 2 * hd
    rows = []
    print(f"{'protocol':<12} {'ms':>10} {'cmp/s':>14} {'kB/party':>10} {'B/cmp':>8}   paper Table 3 (7950X): ms, "
          f"M el/s, kB")
    for v in variants:
        kh, km, _ = P.VARIANT_WIDTHS[v]
        cfg = P.EngineConfig(backend=P.REPLICATED, l=a.length, rotations=1, variant=v)
        sess = P.Session(cfg, master_seed=777)
        hp = P.share_lane_values(dot, kh, rng)
        mp = P.share_lane_values(ml, km, rng) if km else [ml.astype("<u8").view(np.uint8)] * 3
        best, rounds, kb = 1e30, 0, 0.0
        for _ in range(a.repeat):
            sess.comparison_only(hp, mp, n)
            st = sess.last_stats
            best = min(best, st.threshold_ms + st.or_ms)  # device compute, payload upload + parse excluded
            upload = st.prep_ms
            kb = sum(st.lift_bytes[p] + st.msb_bytes[p] for p in range(3)) / 3 / 1000
            rounds = st.lift_rounds + st.msb_rounds
        sess.close()
        name = VARIANT_NAMES[v]
        pt = PAPER_TABLE3[name]
        print(f"{name:<12} {best:>10.3f} {n / (best / 1e3):>14.0f} {kb:>10.1f} {kb * 1000 / n:>8.2f}   "
              f"{pt[0]:>6.2f} {pt[1]:>6.1f} {pt[2]:>6}")
        rows.append({"protocol": name, "comparisons": n, "ms": best, "upload_parse_ms": upload,
                     "throughput_per_s": n / (best / 1e3),
                     "kb_per_party": kb, "bytes_per_comparison": kb * 1000 / n, "rounds": rounds,
                     "paper_table3": {"ms": pt[0], "m_el_per_s": pt[1], "kb_per_party": pt[2]}})
    bits = np.zeros(n, np.uint8)
    if n > 1:
        bits[n // 2] = 1
    sess = P.Session(P.EngineConfig(backend=P.REPLICATED, l=a.length, rotations=1), master_seed=778)
    pay = P.share_bit_words(bits, rng)
    best, kb, rounds = 1e30, 0.0, 0
    for _ in range(a.repeat):
        opened = sess.or_tree_only(pay, n)
        st = sess.last_stats
        best = min(best, st.threshold_ms + st.or_ms)
        kb = (sum(st.or_tree_bytes[p] for p in range(3)) - 2) / 3 / 1000
        rounds = st.or_tree_rounds - 1
    if opened != int(bits.any()):
        raise P.IrisError("or-tree lost the planted bit")
    pt = PAPER_TABLE3["or-tree"]
    print(f"{'or-tree':<12} {best:>10.3f} {n / (best / 1e3):>14.0f} {kb:>10.1f} {kb * 1000 / n:>8.2f}   "
          f"{pt[0]:>6.2f} {pt[1]:>6.1f} {pt[2]:>6}")
    rows.append({"protocol": "or-tree", "comparisons": n, "ms": best, "throughput_per_s": n / (best / 1e3),
                 "kb_per_party": kb, "rounds": rounds,
                 "paper_table3": {"ms": pt[0], "m_el_per_s": pt[1], "kb_per_party": pt[2]}})
    if a.json:
        with open(a.json, "w") as f:
            json.dump(rows, f, indent=2)
            f.write("\n")
    return 0


def cmd_bench(a) -> int:
    """bench --phase full (cmd_bench_full, irismpc_cli.cpp:336-372): a membership query
    of random_record after the DB (Rng(2) stream) against a db_size-row DB dealt with
    seed 900 + r per repetition; best QueryStats.wall_ms (device time here).
    --phase comparison (the default, as in the reference): cmd_bench_comparison."""
    if a.phase == "comparison":
        return cmd_bench_comparison(a)
    if a.phase != "full":
        raise P.ConfigError("--phase must be comparison or full")
    import torch
    backend = BACKENDS[a.backend]
    v = P.MPC_LIFT if a.variant == "all" else P.VARIANTS[a.variant]
    best, last = 1e30, None
    for r in range(a.repeat):
        cfg = P.EngineConfig(backend=backend, l=a.length, rotations=1, variant=v)
        sess = P.Session(cfg, master_seed=900 + r)
        sess.synth_db(a.db_size, rng_seed=2, first=0, mask_density=0.9, deal_seed=900 + r)
        qc, qm = _device_records(sess, 2, a.db_size, 1, 0.9)
        q = [torch.empty(sess.rec, dtype=torch.uint8, device="cuda") for _ in range(3)]
        sess.deal_payload(900 + r, 2, 0, qc, qm, q)
        sess.membership(q)
        st = sess.last_stats
        if st.wall_ms < best:
            best = st.wall_ms
        last = stats_to_json(st, v, backend)
        sess.close()
    print(f"full query: backend={BACKEND_NAMES[backend]} variant={VARIANT_NAMES[v]} s={a.db_size} l={a.length}")
    print(f"  wall {best:.2f} ms, {a.db_size / (best / 1e3):.0f} rows/s")
    pb = last["phase_bytes"]
    print(f"  bytes/party: dot={pb['dot']} lift={pb['lift']} msb={pb['msb']} or_tree={pb['or_tree']}")
    if a.json:
        with open(a.json, "w") as f:
            json.dump(last, f, indent=2)
            f.write("\n")
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="irismpc", description="3-party MPC membership checks on B200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    g = sub.add_parser("gen-db", help="generate a synthetic plaintext iris database")
    g.add_argument("--size", type=int, default=100)
    g.add_argument("--length", type=int, default=12800)
    g.add_argument("--seed", type=int, default=1)
    g.add_argument("--mask-density", type=float, default=0.9, dest="mask_density")
    g.add_argument("--out", required=True)
    s = sub.add_parser("share", help="secret-share a plaintext database (dealer)")
    s.add_argument("--db", required=True)
    s.add_argument("--backend", default="replicated", choices=list(BACKENDS))
    s.add_argument("--variant", default="all")
    s.add_argument("--out-dir", default="shares", dest="out_dir")
    s.add_argument("--seed", type=int, default=1)
    q = sub.add_parser("query", help="share a query and run it against the share directory")
    q.add_argument("--config", default=None)
    q.add_argument("--shares", default=None)
    q.add_argument("--query", required=True)
    q.add_argument("--batch", type=int, default=0)
    q.add_argument("--variant", default="mpc-lift")
    q.add_argument("--stats", default=None)
    q.add_argument("--seed", type=int, default=7)
    q.add_argument("--backend", default="replicated", choices=list(BACKENDS))
    q.add_argument("--length", type=int, default=12800)
    q.add_argument("--match-ratio", type=float, default=0.375, dest="match_ratio")
    q.add_argument("--rotations", type=int, default=31)
    b = sub.add_parser("bench", help="comparison-phase (Table-style) or whole-query benchmark")
    b.add_argument("--phase", default="comparison")
    b.add_argument("--comparisons", type=int, default=100000)
    b.add_argument("--variant", default="all")
    b.add_argument("--backend", default="replicated", choices=list(BACKENDS))
    b.add_argument("--repeat", type=int, default=3)
    b.add_argument("--length", type=int, default=12800)
    b.add_argument("--db-size", type=int, default=1000, dest="db_size")
    b.add_argument("--json", default=None)
    try:
        a = ap.parse_args(argv)
    except SystemExit as e:
        return 0 if e.code == 0 else 2  # flag problems are config errors
    try:
        return {"gen-db": cmd_gen_db, "share": cmd_share, "query": cmd_query, "bench": cmd_bench}[a.cmd](a)
    except P.BoundsError as e:
        print(f"bounds violation: {e}", file=sys.stderr)
        return 4
    except P.DeviceError as e:
        print(f"transport error: {e}", file=sys.stderr)
        return 3
    except P.IrisError as e:
        print(f"error: {e}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
