"""Share / seed / plaintext files (reference io.hpp:28-60, src/io.cpp; §8 f2).

The golden files under tests/golden/files/ were written by the reference itself
(oracle/gen_golden.py -> oracle/_ref: write_iris_db, and the `irismpc share`
dealer's calls deal_seeds / write_seed_file / deal_db_payload / write_share_file,
tools/irismpc_cli.cpp:137-172).  The CPU tests read them with the C-ABI readers,
rewrite them with the C-ABI writers (byte-identical), check the payloads against
the oracle dealer, and check the reference's error cases.  The GPU tests load
the files into HBM with irismpc_gpu_load_db_files and query.
"""
import json
import os
import shutil

import numpy as np
import pytest

import paper_2405_04463_b200 as P
from oracle import pyoracle as O

HERE = os.path.dirname(__file__)
GOLD = json.load(open(os.path.join(HERE, "golden", "ref_vectors.json")))["files"]
FILES = os.path.join(HERE, "golden", "files")


def _f(name):
    return os.path.join(FILES, name)


def _records():
    return O.records(O.Rng(GOLD["records_rng"]), GOLD["l"], GOLD["s"], 0.85)


def test_iris_db_read_and_rewrite(tmp_path):
    codes, masks, l = P.read_iris_db(_f(GOLD["db"]))
    dc, dm = _records()
    assert l == GOLD["l"]
    np.testing.assert_array_equal(codes, dc)
    np.testing.assert_array_equal(masks, dm)
    out = tmp_path / "db.irmp"
    P.write_iris_db(out, codes, masks, l)
    assert out.read_bytes() == open(_f(GOLD["db"]), "rb").read()


@pytest.mark.parametrize("idx", range(len(GOLD["shares"])))
def test_share_files_match_reference_dealer(idx, tmp_path):
    e = GOLD["shares"][idx]
    be, var = e["backend"], e["variant"]
    dc, dm = _records()
    # the dealer's payload = deal_db_payload with Rng(derive(seed_from_u64(seed), variant + 1))
    ref = O.deal(be, GOLD["l"], dc, dm, O.Rng(sub=(GOLD["seed"], var + 1)), variant=var)
    for p, name in enumerate(e["files"]):
        h = P.read_share_header(_f(name))
        assert (h.backend, h.variant, h.party, h.l, h.s) == (be, var, p + 1, GOLD["l"], GOLD["s"])
        raw = open(_f(name), "rb").read()
        assert raw[24:] == ref[p].tobytes()
        out = tmp_path / name
        P.write_share_file(out, be, var, p + 1, GOLD["l"], GOLD["s"], raw[24:])
        assert out.read_bytes() == raw
    # seeds: deal_seeds(Rng(derive(seed_from_u64(seed), 0x5eed))) == run_parties' seeds
    seeds = P.read_seed_files([_f(n) for n in e["seed_files"]])
    assert bytes(seeds) == bytes(O.party_seeds(GOLD["seed"]))
    for p, name in enumerate(e["seed_files"]):
        out = tmp_path / name
        P.write_seed_file(out, p + 1, seeds[16 * p:16 * p + 16], seeds[16 * ((p + 2) % 3):16 * ((p + 2) % 3) + 16])
        assert out.read_bytes() == open(_f(name), "rb").read()


def _corrupt(src, dst, at, value):
    b = bytearray(open(src, "rb").read())
    b[at] = value
    open(dst, "wb").write(bytes(b))


def test_share_header_rejections(tmp_path):
    """read_share_file's errors (io.cpp:125-146): magic, version, width fields, size."""
    src = _f(GOLD["shares"][1]["files"][0])  # Shamir mpc-lift, party 1
    cases = {"magic": (0, ord("X")), "version": (4, 2), "code_k": (8, 32), "mask_k": (9, 0)}
    for name, (at, v) in cases.items():
        dst = tmp_path / f"{name}.irs"
        _corrupt(src, dst, at, v)
        with pytest.raises(P.ConfigError):
            P.read_share_header(dst)
        if O.ref_available():
            assert O.ref_read_share_file(str(dst)) == 2, name
    trunc = tmp_path / "short.irs"
    open(trunc, "wb").write(open(src, "rb").read()[:-1])
    with pytest.raises(P.ConfigError):
        P.read_share_header(trunc)
    if O.ref_available():
        assert O.ref_read_share_file(str(trunc)) == 2
        assert O.ref_read_share_file(src)[:5] == (1, 1, 1, GOLD["l"], GOLD["s"])


def test_seed_file_rejections(tmp_path):
    names = GOLD["shares"][0]["seed_files"]
    paths = [tmp_path / n for n in names]
    for n, p in zip(names, paths):
        shutil.copy(_f(n), p)
    P.read_seed_files(paths)
    # wrong party in file 2
    _corrupt(_f(names[1]), paths[1], 5, 3)
    with pytest.raises(P.ConfigError):
        P.read_seed_files(paths)
    # party 2's prev seed disagrees with party 1's own seed
    shutil.copy(_f(names[1]), paths[1])
    b = bytearray(open(paths[1], "rb").read())
    b[22] ^= 1
    open(paths[1], "wb").write(bytes(b))
    with pytest.raises(P.ConfigError):
        P.read_seed_files(paths)


def test_iris_db_rejections(tmp_path):
    bad = tmp_path / "bad.irmp"
    _corrupt(_f(GOLD["db"]), bad, 0, ord("X"))
    with pytest.raises(P.ConfigError):
        P.read_iris_db(bad)
    trunc = tmp_path / "trunc.irmp"
    open(trunc, "wb").write(open(_f(GOLD["db"]), "rb").read()[:-3])
    with pytest.raises(P.ConfigError):
        P.read_iris_db(trunc)


# ------------------------------------------------------------------ GPU

def _gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a B200")
    return torch


@pytest.mark.gpu
@pytest.mark.parametrize("idx", range(len(GOLD["shares"])))
def test_load_db_files_and_query(idx):
    """Party ingestion: the three IRS1 files + IRSD seeds -> HBM -> membership query == oracle."""
    _gpu()
    e = GOLD["shares"][idx]
    be, var, l = e["backend"], e["variant"], GOLD["l"]
    seeds = P.read_seed_files([_f(n) for n in e["seed_files"]])
    cfg = P.EngineConfig(backend=be, l=l, rotations=1, debug_rows=True, variant=var)
    sess = P.Session(cfg, seeds=seeds)
    sess.load_db_files([_f(n) for n in e["files"]])
    assert sess.s == GOLD["s"]
    dc, dm = _records()
    qc, qm = dc[1:2].copy(), dm[1:2].copy()
    q = O.deal(be, l, qc, qm, O.Rng(sub=(5, 2)), variant=var)
    m = sess.membership(q, want_rows=True)
    db = [np.frombuffer(open(_f(n), "rb").read()[24:], np.uint8) for n in e["files"]]
    ref = O.query(O.make_config(be, l, 0.375, 1, debug_rows=True, variant=var), seeds, db, GOLD["s"], q, 1,
                  membership=True)
    assert m == bool(ref.person_match[0]) == True  # noqa: E712  (row 1 is in the DB)
    np.testing.assert_array_equal(sess.row_bits[:GOLD["s"]], ref.row_bits)


@pytest.mark.gpu
def test_load_db_files_streams_multiple_chunks(tmp_path):
    """A 6000-row l=12800 DB (3 x 307 MB files, > 2 staging chunks) loaded from disk
    gives the same query result as the same payloads loaded from host memory."""
    torch = _gpu()
    l, s, persons, seed = 12800, 6000, 2, 17
    cfg = P.EngineConfig(backend=P.SHAMIR, l=l, rotations=31, debug_rows=True)
    a = P.Session(cfg, master_seed=seed)
    wl = l // 64
    codes = torch.empty((s, wl), dtype=torch.int64, device="cuda")
    masks = torch.empty((s, wl), dtype=torch.int64, device="cuda")
    a.synth_records(2, 0, s, 0.9, codes, masks)
    pay = [torch.empty(s * a.rec, dtype=torch.uint8, device="cuda") for _ in range(3)]
    a.deal_payload(seed, 1, 0, codes, masks, pay)
    host = [p.cpu().numpy() for p in pay]
    paths = [tmp_path / f"db.p{p + 1}.irs" for p in range(3)]
    for p in range(3):
        P.write_share_file(paths[p], P.SHAMIR, P.MPC_LIFT, p + 1, l, s, host[p])
    a.load_db(host, s)
    b = P.Session(cfg, master_seed=seed)
    b.load_db_files(paths)
    qc = torch.empty((2 * persons, wl), dtype=torch.int64, device="cuda")
    qm = torch.empty((2 * persons, wl), dtype=torch.int64, device="cuda")
    a.synth_records(2, 4321, 2 * persons, 0.9, qc, qm)  # record 4321 is DB row 4321: a match
    q = [torch.empty(2 * persons * a.rec, dtype=torch.uint8, device="cuda") for _ in range(3)]
    a.deal_payload(seed, 2, 0, qc, qm, q)
    qh = [x.cpu().numpy() for x in q]
    ma = a.batch_query(qh, persons, want_rows=True)
    mb = b.batch_query(qh, persons, want_rows=True)
    np.testing.assert_array_equal(ma, mb)
    np.testing.assert_array_equal(a.row_bits, b.row_bits)
    assert ma[0] == 1


@pytest.mark.gpu
def test_load_db_files_inconsistent_replicated_shares(tmp_path):
    """load_db_files runs the replicated cross-check (party p's prev == party p-1's own)."""
    _gpu()
    e = [x for x in GOLD["shares"] if x["backend"] == 0][0]
    paths = [tmp_path / n for n in e["files"]]
    for n, p in zip(e["files"], paths):
        open(p, "wb").write(open(_f(n), "rb").read())
    b = bytearray(open(paths[1], "rb").read())
    b[24 + 2] ^= 1  # party 2's first `prev` entry no longer equals party 1's `own`
    open(paths[1], "wb").write(bytes(b))
    seeds = P.read_seed_files([_f(n) for n in e["seed_files"]])
    sess = P.Session(P.EngineConfig(backend=P.REPLICATED, l=GOLD["l"], rotations=1), seeds=seeds)
    with pytest.raises(P.InconsistentShareError):
        sess.load_db_files(paths)
    # a share file of another variant is a config mismatch (irismpc_cli.cpp:211-215)
    other = [x for x in GOLD["shares"] if x["backend"] == 1 and x["variant"] == 0][0]
    sess2 = P.Session(P.EngineConfig(backend=P.SHAMIR, l=GOLD["l"], rotations=1), seeds=seeds)
    with pytest.raises(P.ConfigError):
        sess2.load_db_files([_f(n) for n in other["files"]])


@pytest.mark.gpu
@pytest.mark.parametrize("be", [P.SHAMIR, P.REPLICATED])
def test_plain_mask_unaligned_records(be, tmp_path):
    """plain-mask records of l = 8 are not 16-byte aligned (code 16/32 B + 1 mask byte):
    written to files, loaded, and queried against the oracle."""
    _gpu()
    l, s, seed = 8, 57, 19
    dc, dm = O.records(O.Rng(seed), l, s, 0.9)
    db = O.deal(be, l, dc, dm, O.Rng(sub=(seed, 1)), variant=P.PLAIN_MASK)
    assert (s * O.record_bytes(be, l, P.PLAIN_MASK)) % 16 != 0
    paths = [tmp_path / f"p{p}.irs" for p in (1, 2, 3)]
    for p in range(3):
        P.write_share_file(paths[p], be, P.PLAIN_MASK, p + 1, l, s, db[p])
    seeds = O.party_seeds(seed)
    cfg = P.EngineConfig(backend=be, l=l, rotations=1, debug_rows=True, variant=P.PLAIN_MASK)
    sess = P.Session(cfg, seeds=seeds)
    sess.load_db_files(paths)
    qc, qm = dc[5:6].copy(), dm[5:6].copy()
    q = O.deal(be, l, qc, qm, O.Rng(sub=(seed, 2)), variant=P.PLAIN_MASK)
    m = sess.membership(q, want_rows=True)
    ref = O.query(O.make_config(be, l, 0.375, 1, debug_rows=True, variant=P.PLAIN_MASK), seeds, db, s, q, 1,
                  membership=True)
    assert m == bool(ref.person_match[0])
    np.testing.assert_array_equal(sess.row_bits[:s], ref.row_bits)
