"""The `irismpc` CLI on the B200 path (paper_2405_04463_b200/cli.py) vs the
reference's commands (tools/irismpc_cli.cpp; §8 f4): identical files from
gen-db / share, the same query answers and stats JSON schema, the same exit codes."""
import json
import os

import numpy as np
import pytest

import paper_2405_04463_b200 as P
from paper_2405_04463_b200 import cli
from oracle import pyoracle as O


def test_exit_codes_without_gpu(tmp_path):
    # flag problems and config errors are 2 (irismpc_cli.cpp:543-568)
    assert cli.main(["query", "--bogus"]) == 2
    q = tmp_path / "q.irmp"
    dc, dm = O.records(O.Rng(3), 64, 1, 0.9)
    P.write_iris_db(q, dc, dm, 64)
    assert cli.main(["query", "--shares", str(tmp_path / "none"), "--query", str(q), "--length", "64"]) == 2
    assert cli.main(["query", "--shares", str(tmp_path), "--query", str(q), "--length", "128"]) == 2
    assert cli.main(["bench", "--phase", "bogus"]) == 2


def _gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a B200")


@pytest.mark.gpu
def test_gen_db_matches_reference_records(tmp_path):
    _gpu()
    out = tmp_path / "db.irmp"
    assert cli.main(["gen-db", "--size", "7", "--length", "256", "--seed", "5", "--out", str(out)]) == 0
    dc, dm = O.records(O.Rng(5), 256, 7, 0.9)  # random_record(l, Rng(seed), 0.9), pinned to the reference
    ref = tmp_path / "ref.irmp"
    P.write_iris_db(ref, dc, dm, 256)  # byte-identical to the reference writer (test_files.py)
    assert out.read_bytes() == ref.read_bytes()


@pytest.mark.gpu
@pytest.mark.parametrize("backend", ["replicated", "shamir-galois"])
def test_share_matches_reference_dealer(tmp_path, backend):
    _gpu()
    l, s, seed = 128, 9, 11
    dc, dm = O.records(O.Rng(4), l, s, 0.85)
    db = tmp_path / "db.irmp"
    P.write_iris_db(db, dc, dm, l)
    out = tmp_path / "shares"
    assert cli.main(["share", "--db", str(db), "--backend", backend, "--variant", "all", "--out-dir", str(out),
                     "--seed", str(seed)]) == 0
    be = cli.BACKENDS[backend]
    seeds = P.read_seed_files([cli.seed_path(out, p) for p in (1, 2, 3)])
    assert bytes(seeds) == bytes(O.party_seeds(seed))
    for v in (P.PLAIN_MASK, P.MPC_LIFT, P.CONST_LIFT, P.NO_LIFT):
        ref = O.deal(be, l, dc, dm, O.Rng(sub=(seed, v + 1)), variant=v)
        for p in range(3):
            raw = open(cli.share_path(out, v, p + 1), "rb").read()
            h = P.read_share_header(cli.share_path(out, v, p + 1))
            assert (h.backend, h.variant, h.party, h.l, h.s) == (be, v, p + 1, l, s)
            assert raw[24:] == ref[p].tobytes()
        if O.ref_available():  # the reference's own dealer writes the same bytes
            rp = [str(tmp_path / f"r{v}.p{p}.irs") for p in (1, 2, 3)]
            rs = [str(tmp_path / f"r{v}.p{p}.irsd") for p in (1, 2, 3)]
            O.ref_share_files(str(db), be, v, seed, rp, rs)
            for p in range(3):
                assert open(rp[p], "rb").read() == open(cli.share_path(out, v, p + 1), "rb").read()
                assert open(rs[p], "rb").read() == open(cli.seed_path(out, p + 1), "rb").read()


@pytest.mark.gpu
def test_query_all_variants_and_stats(tmp_path, capsys):
    _gpu()
    l, s, persons, seed, qseed = 256, 40, 2, 13, 21
    dc, dm = O.records(O.Rng(6), l, s, 0.85)
    db = tmp_path / "db.irmp"
    P.write_iris_db(db, dc, dm, l)
    out = tmp_path / "shares"
    assert cli.main(["share", "--db", str(db), "--backend", "shamir-galois", "--out-dir", str(out),
                     "--seed", str(seed)]) == 0
    qc, qm = O.records(O.Rng(7), l, 2 * persons, 0.85)
    qc[2], qm[2] = dc[17], dm[17]  # person 1's left eye is DB row 17
    qf = tmp_path / "q.irmp"
    P.write_iris_db(qf, qc, qm, l)
    st = tmp_path / "stats.json"
    capsys.readouterr()
    rc = cli.main(["query", "--shares", str(out), "--query", str(qf), "--batch", str(persons), "--variant", "all",
                   "--stats", str(st), "--seed", str(qseed), "--backend", "shamir-galois", "--length", str(l),
                   "--rotations", "5"])
    assert rc == 0
    lines = capsys.readouterr().out.splitlines()
    assert lines[:3] == ["variant mpc-lift: false true", "variant const-lift: false true",
                         "variant no-lift: false true"]
    assert lines[3] == "all variants agree"
    stats = json.load(open(st))
    assert [x["variant"] for x in stats] == ["mpc-lift", "const-lift", "no-lift"]
    assert set(stats[0]) == {"variant", "backend", "s", "l", "batch", "phase_bytes", "rounds", "wall_ms"}
    assert stats[0]["backend"] == "shamir-galois" and stats[0]["s"] == s and stats[0]["batch"] == persons
    # mpc-lift answer and ledger == the oracle on the same share files and query dealing
    seeds = P.read_seed_files([cli.seed_path(out, p) for p in (1, 2, 3)])
    dbp = [np.frombuffer(open(cli.share_path(out, P.MPC_LIFT, p), "rb").read()[24:], np.uint8) for p in (1, 2, 3)]
    q = O.deal(P.SHAMIR, l, qc, qm, O.Rng(sub=(qseed, 0x9E + P.MPC_LIFT)), variant=P.MPC_LIFT)
    ref = O.query(O.make_config(P.SHAMIR, l, 0.375, 5), seeds, dbp, s, q, persons)
    assert [int(x) for x in ref.person_match] == [0, 1]
    assert stats[0]["phase_bytes"]["dot"] == ref.stats[0]["dot_bytes"]
    assert stats[0]["rounds"]["or_tree"] == ref.stats[0]["or_tree_rounds"]


@pytest.mark.gpu
def test_bench_full(tmp_path, capsys):
    _gpu()
    js = tmp_path / "b.json"
    assert cli.main(["bench", "--phase", "full", "--db-size", "3000", "--repeat", "2", "--backend",
                     "shamir-galois", "--json", str(js)]) == 0
    out = capsys.readouterr().out
    assert out.startswith("full query: backend=shamir-galois variant=mpc-lift s=3000 l=12800")
    d = json.load(open(js))
    assert d["s"] == 3000 and d["phase_bytes"]["dot"] == 4 * 3000 and d["rounds"]["msb"] == 31


@pytest.mark.gpu
def test_query_with_reference_config_json(tmp_path, capsys):
    """`query --config` reads the reference's party config (share_dir, backend, l,
    match_ratio, rotations; endpoints ignored) and answers a membership query."""
    _gpu()
    l, s, seed = 128, 25, 3
    dc, dm = O.records(O.Rng(8), l, s, 0.9)
    db = tmp_path / "db.irmp"
    P.write_iris_db(db, dc, dm, l)
    out = tmp_path / "shares"
    assert cli.main(["share", "--db", str(db), "--backend", "replicated", "--variant", "mpc-lift",
                     "--out-dir", str(out), "--seed", str(seed)]) == 0
    cfg = tmp_path / "p1.json"
    cfg.write_text(json.dumps({"party": 1, "endpoints": ["127.0.0.1:1", "127.0.0.1:2", "127.0.0.1:3"],
                               "backend": "replicated", "l": l, "match_ratio": 0.375, "rotations": 1,
                               "share_dir": str(out)}))
    q = tmp_path / "q.irmp"
    P.write_iris_db(q, dc[11:12], dm[11:12], l)
    capsys.readouterr()
    assert cli.main(["query", "--config", str(cfg), "--query", str(q)]) == 0
    assert capsys.readouterr().out.splitlines()[0] == "variant mpc-lift: true"


@pytest.mark.gpu
def test_bench_comparison_table(tmp_path, capsys):
    """`bench` (default --phase comparison, irismpc_cli.cpp:373-458): one row per
    variant plus the OR-tree row; kB/party equals the reference's acceptance
    ledger (proj/test_output.txt:17-21)."""
    _gpu()
    js = tmp_path / "c.json"
    assert cli.main(["bench", "--repeat", "2", "--json", str(js)]) == 0
    out = capsys.readouterr().out.splitlines()
    assert out[0].split()[:5] == ["protocol", "ms", "cmp/s", "kB/party", "B/cmp"]
    rows = {r["protocol"]: r for r in json.load(open(js))}
    assert set(rows) == {"plain-mask", "mpc-lift", "const-lift", "no-lift", "or-tree"}
    assert rows["plain-mask"]["kb_per_party"] == pytest.approx(362.50)
    assert rows["mpc-lift"]["kb_per_party"] == pytest.approx(2095.8333, abs=1e-3)
    assert rows["const-lift"]["kb_per_party"] == pytest.approx(762.50)
    assert rows["no-lift"]["kb_per_party"] == pytest.approx(762.50)
    assert rows["or-tree"]["kb_per_party"] == pytest.approx(12.5087, abs=1e-3)
