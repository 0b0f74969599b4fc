"""The oracle (C restatement) pinned against the reference's golden vectors.

Expectations in tests/golden/ref_vectors.json were produced by the reference
itself (oracle/gen_golden.py over oracle/_ref).  When oracle/_ref is present
(this container), the restatement is additionally diffed live against it.
"""
import hashlib
import json
import os

import numpy as np
import pytest

from oracle import pyoracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "ref_vectors.json")))


def _sha(a):
    """gen_golden.sha: little-endian bytes at the array's ring width."""
    dt = {np.dtype(np.uint16): "<u2", np.dtype(np.uint32): "<u4", np.dtype(np.int64): "<i8"}[a.dtype]
    return hashlib.sha256(np.ascontiguousarray(a).astype(dt).tobytes()).hexdigest()


def test_prf_kats():
    g = GOLD["prf"]
    s42 = O.seed_from_u64(42)
    assert bytes(s42).hex() == g["seed_from_u64_42"]
    # seed_from_u64(42) KAT recorded from the reference
    assert bytes(s42).hex() == "0dc1b79bfd711811bff2b5d48d0deeb1"
    assert [int(x) for x in O.chacha_block(s42, 0)] == g["chacha12_seed42_block0_stream0"]
    assert [int(x) for x in O.chacha_block(s42, 5, 3)] == g["chacha12_seed42_block5_stream3"]
    b = O.chacha_block(s42, 0)
    first = [int(b[2 * i]) | (int(b[2 * i + 1]) << 32) for i in range(4)]
    assert first == [0x402777fd6e386d1e, 0xc496c74fbbc0672a, 0xb725cec52db6ca88, 0xdeb6c2f8c503aa7e]
    assert bytes(O.party_seeds(7)).hex() == g["party_seeds_7"]
    r = O.Rng(2)
    assert [str(r.next()) for _ in range(20)] == g["rng2_first20"]


def test_galois_lambda():
    lam = O.lambda16()
    assert [int(x) for x in lam] == GOLD["lambda16"]
    # closed forms (test_galois.cpp:113-115): 1+2X, -(1+2X), 1
    assert [int(x) for x in lam] == [1, 2, 0xFFFF, 0xFFFE, 1, 0]
    # the 32-bit lambdas used by const-lift / no-lift: same closed forms mod 2^32
    assert [int(x) for x in O.lambda_k(32)] == [1, 2, 0xFFFFFFFF, 0xFFFFFFFE, 1, 0]
    assert [int(x) for x in O.lambda_k(32)] == GOLD["lambda32_restated"]


def test_random_records():
    g = GOLD["random_records_rng11_l128"]
    rng = O.Rng(11)
    for i, d in enumerate(g["density"]):
        c, m = rng.record(128, d)
        assert [str(int(w)) for w in c] == g["code"][i]
        assert [str(int(w)) for w in m] == g["mask"][i]


@pytest.mark.parametrize("idx", range(len(GOLD["deal"])))
def test_dealer(idx):
    d = GOLD["deal"][idx]
    dc, dm = O.records(O.Rng(d["records_rng"]), d["l"], d["nrec"], 0.9)
    var = d.get("variant", O.MPC_LIFT)
    pay = O.deal(d["backend"], d["l"], dc, dm, O.Rng(sub=(d["deal_seed"], d["tag"])), variant=var)
    assert [hashlib.sha256(p.tobytes()).hexdigest() for p in pay] == d["sha256"]


def _case_inputs(c):
    rng = O.Rng(c["seed"])
    dc, dm = O.records(rng, c["l"], c["s"], 0.85)
    nq = 1 if c["membership"] else 2 * c["persons"]
    qc, qm = O.records(rng, c["l"], nq, 0.85)
    if c["planted"] and c["s"] > 0:
        qc[0] = dc[c["s"] // 2]
        qm[0] = dm[c["s"] // 2]
    return dc, dm, qc, qm


@pytest.mark.parametrize("idx", range(len(GOLD["cases"])))
def test_protocol_golden(idx):
    c = GOLD["cases"][idx]
    dc, dm, qc, qm = _case_inputs(c)
    var = c.get("variant", O.MPC_LIFT)
    cfg = O.make_config(c["backend"], c["l"], c["ratio"], c["rotations"], debug_rows=True, variant=var)
    res = O.run_local(cfg, c["seed"], dc, dm, qc, qm, c["persons"], c["membership"], want_all=True)
    n = c["lanes"]
    assert res.row_bits.size == n
    assert [int(x) for x in res.person_match] == c["person_match"]
    assert np.packbits(res.row_bits, bitorder="little").tobytes().hex() == c["row_bits_hex"]
    assert res.stats == c["stats"]
    assert _sha(res.dot_hd) == c["sha256"]["dot_hd"]        # L1
    assert _sha(res.rs_hd) == c["sha256"]["rs_hd"]          # L2
    kc = O.cmp_bits(var)
    dsum = res.diff.astype(np.uint64).sum(0) & ((1 << kc) - 1)
    assert (((dsum >> (kc - 1)) & 1).astype(np.uint8) == res.row_bits).all()
    assert ((res.msb[0] ^ res.msb[1] ^ res.msb[2]) == res.row_bits).all()
    if var != O.MPC_LIFT:
        if O.mask_bits(var):
            assert _sha(res.dot_ml) == c["sha256"]["dot_ml"]
            assert _sha(res.rs_ml) == c["sha256"]["rs_ml"]
        else:
            assert _sha(res.public_ml) == c["sha256"]["public_ml"]
        return
    assert _sha(res.dot_ml) == c["sha256"]["dot_ml"]
    assert _sha(res.rs_ml) == c["sha256"]["rs_ml"]
    # L3: reconstructed distances are the plaintext masked dot and mask length
    rec_hd = (res.rs_hd.astype(np.uint32).sum(0) & 0xFFFF)
    rec_ml = (res.rs_ml.astype(np.uint32).sum(0) & 0xFFFF)
    assert ((res.dot_hd.astype(np.uint32).sum(0) & 0xFFFF) == rec_hd).all()
    assert ((res.dot_ml.astype(np.uint32).sum(0) & 0xFFFF) == rec_ml).all()
    # lift: reconstructed ml32 == ml; diff sign == row bit
    assert ((res.ml32.astype(np.uint64).sum(0) & 0xFFFFFFFF) == rec_ml).all()
    d32 = (res.diff.astype(np.uint64).sum(0) & 0xFFFFFFFF)
    assert (((d32 >> 31) & 1).astype(np.uint8) == res.row_bits).all()
    assert ((res.msb[0] ^ res.msb[1] ^ res.msb[2]) == res.row_bits).all()


def _plain_counts(qc, qm, dc, dm, l):
    """oracle.hpp:35-44 count_pair over unpacked bits."""
    def bits(w):
        return np.unpackbits(w.view(np.uint8), bitorder="little")[:l].astype(bool)
    qcb, qmb, dcb, dmb = bits(qc), bits(qm), bits(dc), bits(dm)
    m = qmb & dmb
    return int((m & (qcb != dcb)).sum()), int(m.sum())


def test_reconstructed_distances_match_plaintext():
    # membership, l=64: lanes are DB rows; rs reconstructs to ml - 2*hd and ml
    c = GOLD["cases"][4]
    dc, dm, qc, qm = _case_inputs(c)
    cfg = O.make_config(c["backend"], c["l"], c["ratio"], 1, debug_rows=True)
    res = O.run_local(cfg, c["seed"], dc, dm, qc, qm, 1, True, want_all=True)
    a, b = cfg.a, cfg.b
    for row in range(c["s"]):
        hd, ml = _plain_counts(qc[0], qm[0], dc[row], dm[row], c["l"])
        dot = ml - 2 * hd
        assert int(res.rs_hd[:, row].astype(np.uint32).sum() & 0xFFFF) == dot & 0xFFFF
        assert int(res.rs_ml[:, row].astype(np.uint32).sum() & 0xFFFF) == ml
        assert bool(res.row_bits[row]) == (b * dot > a * ml)   # oracle.hpp:49-57


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built (no /root/reference here)")
@pytest.mark.parametrize("var", [O.PLAIN_MASK, O.CONST_LIFT, O.NO_LIFT])
@pytest.mark.parametrize("be", [0, 1])
def test_variant_restatement_vs_live_reference(var, be):
    rng = O.Rng(3000 + var)
    l, s, persons, r = 128, 6, 3, 3
    dc, dm = O.records(rng, l, s, 0.85)
    qc, qm = O.records(rng, l, 2 * persons, 0.85)
    qc[2] = dc[4]
    qm[2] = dm[4]
    cfg = O.make_config(be, l, 0.375, r, debug_rows=True, variant=var)
    a = O.run_local(cfg, 9, dc, dm, qc, qm, persons, want_all=True)
    b = O.ref_run_local(be, l, 0.375, r, 9, dc, dm, qc, qm, persons, debug_rows=True, variant=var)
    assert (a.person_match == b["person_match"]).all()
    assert (a.row_bits == b["row_bits"]).all()
    assert a.stats == b["stats"]
    db = O.deal(be, l, dc, dm, O.Rng(sub=(9, 1)), variant=var)
    q = O.deal(be, l, qc, qm, O.Rng(sub=(9, 2)), variant=var)
    dh, dmm, rh, rm = O.ref_dots_reshare(be, l, r, O.party_seeds(9), db, s, q, persons, variant=var)
    assert (dh == a.dot_hd).all() and (rh == a.rs_hd).all()
    if O.mask_bits(var):
        assert (dmm == a.dot_ml).all() and (rm == a.rs_ml).all()
    else:
        assert (O.ref_dots_reshare.public_ml == a.public_ml).all()


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built (no /root/reference here)")
@pytest.mark.parametrize("be", [0, 1])
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_restatement_vs_live_reference(be, seed):
    rng = O.Rng(1000 + seed)
    l, s, persons, r = 256, 5, 3, 3
    dc, dm = O.records(rng, l, s, 0.85)
    qc, qm = O.records(rng, l, 2 * persons, 0.85)
    qc[3] = dc[1]
    qm[3] = dm[1]
    cfg = O.make_config(be, l, 0.375, r, debug_rows=True)
    a = O.run_local(cfg, seed, dc, dm, qc, qm, persons)
    b = O.ref_run_local(be, l, 0.375, r, seed, dc, dm, qc, qm, persons, debug_rows=True)
    assert (a.person_match == b["person_match"]).all()
    assert (a.row_bits == b["row_bits"]).all()
    assert a.stats == b["stats"]


def test_stream_positions_match_reference_draw_counts():
    # draws = 2n + 125W + OR words (+2n seed1, +6n seed3)
    c = GOLD["cases"][10]
    dc, dm, qc, qm = _case_inputs(c)
    cfg = O.make_config(c["backend"], c["l"], c["ratio"], c["rotations"])
    res = O.run_local(cfg, c["seed"], dc, dm, qc, qm, c["persons"], c["membership"])
    n = c["lanes"]
    W = (n + 63) // 64
    p1, p2, p3 = (int(x) for x in res.stream_pos)
    assert p1 - p2 == 2 * n and p3 - p2 == 6 * n
    assert p2 >= 2 * n + 125 * W
