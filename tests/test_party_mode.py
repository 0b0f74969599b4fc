"""Party mode: one party per context, every reference message
through a transport.  Here the three parties run on one GPU in three host
threads over the in-process mailbox (InProcNet); tests/test_party_nccl.py runs
them as three NCCL ranks on three GPUs.

Each party's (own, prev) shares are compared with components (p, p-1) of the
oracle's component-form run, the measured ledger with the reference's
QueryStats, and the stream positions with the reference's draw counts.
"""
import numpy as np
import pytest

import paper_2405_04463_b200 as P
from oracle import pyoracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a B200", allow_module_level=True)


def _case(be, l, s, persons, r, seed, membership=False, density=0.9):
    rng = O.Rng(seed)
    dc, dm = O.records(rng, l, s, density)
    nq = 1 if membership else 2 * persons
    qc, qm = O.records(rng, l, nq, density)
    if s:
        qc[0], qm[0] = dc[s // 2], dm[s // 2]
    db = O.deal(be, l, dc, dm, O.Rng(sub=(seed, 1)))
    q = O.deal(be, l, qc, qm, O.Rng(sub=(seed, 2)))
    return db, q


@pytest.mark.parametrize("be,l,s,persons,r,seed", [
    (O.SHAMIR, 256, 300, 3, 5, 71),
    (O.REPLICATED, 256, 130, 2, 31, 72),
    (O.SHAMIR, 12800, 64, 2, 31, 73),
    (O.REPLICATED, 128, 0, 4, 3, 74),   # pairs only
])
def test_party_mode_shares_ledger_positions(be, l, s, persons, r, seed):
    db, q = _case(be, l, s, persons, r, seed)
    seeds = O.party_seeds(seed)
    cfg = P.EngineConfig(backend=be, l=l, rotations=r, debug_rows=True)
    parties = P.run_parties_inproc(cfg, seeds, db, s, q, persons, want_rows=True)
    ref = O.query(O.make_config(be, l, 0.375, r, debug_rows=True), seeds, db, s, q, persons, want_all=True)
    n = P.lane_count(persons, s, r)
    np.testing.assert_array_equal(parties[0].result, ref.person_match)            # L5 at P1
    np.testing.assert_array_equal(parties[0].row_bits[:n], ref.row_bits)          # L4 at P1
    for i, pt in enumerate(parties):
        own, prev = i, (i + 2) % 3
        np.testing.assert_array_equal(pt.read_tap(P.TAP_DOT_HD, n), ref.dot_hd[own], err_msg=f"P{i+1} dot_hd")
        np.testing.assert_array_equal(pt.read_tap(P.TAP_DOT_ML, n), ref.dot_ml[own], err_msg=f"P{i+1} dot_ml")
        for tap, name in ((P.TAP_RS_HD, "rs_hd"), (P.TAP_RS_ML, "rs_ml"), (P.TAP_ML32, "ml32"),
                          (P.TAP_DIFF, "diff"), (P.TAP_MSB, "msb")):
            got = pt.read_tap(tap, n)
            want = getattr(ref, name)
            np.testing.assert_array_equal(got[0], want[own], err_msg=f"P{i+1} {name} own")
            np.testing.assert_array_equal(got[1], want[prev], err_msg=f"P{i+1} {name} prev")
        assert pt.last_stats.ledger() == ref.stats[i], f"P{i+1} ledger"
        np.testing.assert_array_equal(pt.stream_positions(), [ref.stream_pos[own], ref.stream_pos[prev]])


@pytest.mark.parametrize("be", [O.SHAMIR, O.REPLICATED])
def test_party_mode_membership(be):
    l, s, seed = 128, 500, 75
    db, q = _case(be, l, s, 1, 1, seed, membership=True)
    seeds = O.party_seeds(seed)
    cfg = P.EngineConfig(backend=be, l=l, rotations=1, debug_rows=True)
    parties = P.run_parties_inproc(cfg, seeds, db, s, q, membership=True, want_rows=True)
    ref = O.query(O.make_config(be, l, 0.375, 1, debug_rows=True), seeds, db, s, q, 1, membership=True)
    assert parties[0].result == bool(ref.person_match[0]) is True
    np.testing.assert_array_equal(parties[0].row_bits[:s], ref.row_bits)
    for i, pt in enumerate(parties):
        assert pt.last_stats.ledger() == ref.stats[i]


def test_party_mode_matches_single_context_engine():
    """The party-split run and the fused 3-party engine give the same bits at a
    configs[1]-like batch (16 persons, 31 rotations)."""
    be, l, s, persons, r, seed = O.SHAMIR, 12800, 2000, 16, 31, 76
    db, q = _case(be, l, s, persons, r, seed)
    seeds = O.party_seeds(seed)
    cfg = P.EngineConfig(backend=be, l=l, rotations=r)
    parties = P.run_parties_inproc(cfg, seeds, db, s, q, persons)
    sess = P.Session(cfg, seeds=seeds)
    sess.load_db(db, s)
    m = sess.batch_query(q, persons)
    np.testing.assert_array_equal(parties[0].result, m)
    assert m[0] == 1


@pytest.mark.parametrize("be", [O.SHAMIR, O.REPLICATED])
def test_empty_db_membership_both_engines(be):
    """s = 0: zero lanes, every round still runs (empty messages); no match, and
    the ledger equals the reference's (oracle pinned to the live reference)."""
    l, seed = 128, 77
    rng = O.Rng(seed)
    qc, qm = O.records(rng, l, 1, 0.9)
    q = O.deal(be, l, qc, qm, O.Rng(sub=(seed, 2)))
    db = [np.zeros(0, np.uint8)] * 3
    seeds = O.party_seeds(seed)
    cfg = P.EngineConfig(backend=be, l=l, rotations=1)
    ref = O.query(O.make_config(be, l, 0.375, 1), seeds, db, 0, q, 1, membership=True)
    assert int(ref.person_match[0]) == 0
    parties = P.run_parties_inproc(cfg, seeds, db, 0, q, membership=True)
    assert parties[0].result is False
    for i, pt in enumerate(parties):
        assert pt.last_stats.ledger() == ref.stats[i]
    sess = P.Session(cfg, seeds=seeds)
    sess.load_db(db, 0)
    assert sess.membership(q) is False
    np.testing.assert_array_equal(sess.stream_positions(), ref.stream_pos)


@pytest.mark.parametrize("var", [P.PLAIN_MASK, P.CONST_LIFT, P.NO_LIFT])
@pytest.mark.parametrize("be,l,s,persons,r,seed", [
    (O.SHAMIR, 256, 300, 3, 5, 81),
    (O.REPLICATED, 128, 90, 2, 31, 82),
    (O.SHAMIR, 12800, 40, 2, 31, 83),
])
def test_party_mode_variants(var, be, l, s, persons, r, seed):
    """Party mode for plain-mask / const-lift / no-lift: shares through the MSB,
    ledger, stream positions, row and person bits vs the oracle."""
    rng = O.Rng(seed)
    dc, dm = O.records(rng, l, s, 0.9)
    qc, qm = O.records(rng, l, 2 * persons, 0.9)
    qc[0], qm[0] = dc[s // 2], dm[s // 2]
    db = O.deal(be, l, dc, dm, O.Rng(sub=(seed, 1)), variant=var)
    q = O.deal(be, l, qc, qm, O.Rng(sub=(seed, 2)), variant=var)
    seeds = O.party_seeds(seed)
    cfg = P.EngineConfig(backend=be, l=l, rotations=r, debug_rows=True, variant=var)
    parties = P.run_parties_inproc(cfg, seeds, db, s, q, persons, want_rows=True)
    ref = O.query(O.make_config(be, l, 0.375, r, debug_rows=True, variant=var), seeds, db, s, q, persons,
                  want_all=True)
    n = P.lane_count(persons, s, r)
    np.testing.assert_array_equal(parties[0].result, ref.person_match)
    np.testing.assert_array_equal(parties[0].row_bits[:n], ref.row_bits)
    assert parties[0].result[0] == 1
    for i, pt in enumerate(parties):
        own, prev = i, (i + 2) % 3
        np.testing.assert_array_equal(pt.read_tap(P.TAP_DOT_HD, n), ref.dot_hd[own], err_msg=f"P{i+1} dot_hd")
        if P.VARIANT_WIDTHS[var][1]:
            np.testing.assert_array_equal(pt.read_tap(P.TAP_DOT_ML, n), ref.dot_ml[own], err_msg=f"P{i+1} dot_ml")
        else:
            np.testing.assert_array_equal(pt.read_tap(P.TAP_DOT_ML, n), ref.public_ml, err_msg=f"P{i+1} public_ml")
        for tap, name in ((P.TAP_RS_HD, "rs_hd"), (P.TAP_RS_ML, "rs_ml"), (P.TAP_ML32, "ml32"),
                          (P.TAP_DIFF, "diff"), (P.TAP_MSB, "msb")):
            got = pt.read_tap(tap, n)
            want = getattr(ref, name)
            np.testing.assert_array_equal(got[0], want[own], err_msg=f"P{i+1} {name} own")
            np.testing.assert_array_equal(got[1], want[prev], err_msg=f"P{i+1} {name} prev")
        assert pt.last_stats.ledger() == ref.stats[i], f"P{i+1} ledger"
        np.testing.assert_array_equal(pt.stream_positions(), [ref.stream_pos[own], ref.stream_pos[prev]])
