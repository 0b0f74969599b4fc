"""The reference's own edge-case families through the B200 (the acceptance-C1
equivalent): every instance of tests/golden/equiv_grid.npz -- the randomized
equivalence grid of equiv_common.hpp:59-146 (both backends x 4 variants x
l in {8, 64, 128} x s in {1, 4, 64}, mask densities {0, 1, 0.3, 0.85},
planted noisy copies; ratios 0.375 and 0.3), the 100 threshold-boundary
instances b*dot in {a*ml - 1, a*ml, a*ml + 1}, and test_engine.cpp's planted
self-match, complement row and ml = 0 cases -- runs as a 3-party membership
query on the GPU.  The opened aggregate must equal the reference's plaintext
oracle (and the reference's own 3-party result), and every opened debug row
bit must equal the plaintext per-row predicate.  Also the l = 12800
all-variant case of test_equivalence.cpp:35-51 and configs[0] at its exact
shape, share for share."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a B200", allow_module_level=True)

import paper_2405_04463_b200 as P  # noqa: E402
from oracle import pyoracle as O  # noqa: E402
from equiv_grid import load, plain_bits  # noqa: E402

INST = load()
GROUPS = sorted({(x["backend"], x["variant"], x["l"], x["ratio"]) for x in INST})


@pytest.mark.parametrize("be,var,l,ratio", GROUPS)
def test_equivalence_grid_on_gpu(be, var, l, ratio):
    cfg = P.EngineConfig(backend=be, l=l, match_ratio=ratio, rotations=1, debug_rows=True, variant=var)
    sess = P.Session(cfg, master_seed=1)
    bad = []
    n = 0
    for x in INST:
        if (x["backend"], x["variant"], x["l"], x["ratio"]) != (be, var, l, ratio):
            continue
        n += 1
        db = P._dealt_on_device(sess, x["db_codes"], x["db_masks"], x["seed"], 1)
        sess.load_db(db, x["s"])
        q = P._dealt_on_device(sess, x["q_code"], x["q_mask"], x["seed"], 2)
        sess.set_stream_positions([0, 0, 0])  # run_membership_local starts every stream at 0
        got = int(sess.membership(q, want_rows=True))
        rows = sess.row_bits[:x["s"]]
        want_rows = plain_bits(x)
        if got != x["want"] or not np.array_equal(rows, want_rows) or (
                x["kind"] == "grid" and not np.array_equal(rows, x["ref_row_bits"])):
            bad.append((x["kind"], x["s"], x["seed"], got, x["want"]))
    assert n > 0
    assert not bad, f"{len(bad)} of {n} instances differ: {bad[:5]}"


@pytest.mark.parametrize("var", [P.PLAIN_MASK, P.MPC_LIFT, P.CONST_LIFT, P.NO_LIFT])
@pytest.mark.parametrize("be", [O.REPLICATED, O.SHAMIR])
def test_paper_scale_length_all_variants(be, var):
    """test_equivalence.cpp:35-51: l = 12800, 4 rows, query = row 1 with every
    5th code bit flipped (close to, not equal to the row), vs the oracle; plus
    the same query against the reference's own 3-party run."""
    l = 12800
    rng = O.Rng(4242)
    dc, dm = O.records(rng, l, 4, 0.9)
    qc, qm = dc[1:2].copy(), dm[1:2].copy()
    bits = np.unpackbits(qc.view(np.uint8), bitorder="little")
    bits[::5] ^= 1
    qc = np.packbits(bits, bitorder="little").view(np.uint64).reshape(1, -1)
    cfg = P.EngineConfig(backend=be, l=l, rotations=1, debug_rows=True, variant=var)
    m, sess = P.run_batch_local(cfg, qc, qm, dc, dm, 4242, membership=True, want_rows=True)
    inst = dict(l=l, s=4, ratio=0.375, variant=var, q_code=qc, q_mask=qm, db_codes=dc, db_masks=dm)
    want_rows = plain_bits(inst)
    np.testing.assert_array_equal(sess.row_bits[:4], want_rows)
    assert int(m[0]) == int(want_rows.any())
    if O.ref_available():
        ref = O.ref_run_local(be, l, 0.375, 1, 4242, dc, dm, qc, qm, 1, membership=True, debug_rows=True,
                              variant=var)
        assert int(ref["person_match"][0]) == int(m[0])
        np.testing.assert_array_equal(ref["row_bits"], sess.row_bits[:4])


@pytest.mark.parametrize("be", [O.SHAMIR, O.REPLICATED])
def test_configs0_exact_shape_share_for_share(be):
    """BASELINE configs[0] at its exact shape: 1 person (2 eye codes) x 31
    rotations vs a 10,000-row DB, l = 12800, mpc-lift.  Per-party dots (L1) and
    reshared components (L2) equal the REFERENCE's (oracle/_ref), lift / diff /
    MSB components equal the C restatement's, and the opened row bits, person
    bit, ledgers and stream positions equal the reference's run_batch_local."""
    if not O.ref_available():
        pytest.skip("oracle/_ref not shipped")
    l, s, persons, r, seed = 12800, 10_000, 1, 31, 7
    rng = O.Rng(2)
    dc, dm = O.records(rng, l, s, 0.9)
    qc, qm = O.records(rng, l, 2, 0.9)
    qc[0], qm[0] = dc[s // 2], dm[s // 2]
    cfg = P.EngineConfig(backend=be, l=l, rotations=r, debug_rows=True)
    m, sess = P.run_batch_local(cfg, qc, qm, dc, dm, seed, persons=persons, want_rows=True, taps=True)
    n = P.lane_count(persons, s, r)
    db = O.deal(be, l, dc, dm, O.Rng(sub=(seed, 1)))
    q = O.deal(be, l, qc, qm, O.Rng(sub=(seed, 2)))
    r_hd, r_ml, r_rs_hd, r_rs_ml = O.ref_dots_reshare(be, l, r, O.party_seeds(seed), db, s, q, persons)
    np.testing.assert_array_equal(sess.read_tap(P.TAP_DOT_HD, n), r_hd)
    np.testing.assert_array_equal(sess.read_tap(P.TAP_DOT_ML, n), r_ml)
    np.testing.assert_array_equal(sess.read_tap(P.TAP_RS_HD, n), r_rs_hd)
    np.testing.assert_array_equal(sess.read_tap(P.TAP_RS_ML, n), r_rs_ml)
    orc = O.query(O.make_config(be, l, 0.375, r, debug_rows=True), O.party_seeds(seed), db, s, q, persons,
                  want_all=True)
    for k, t in (("ml32", P.TAP_ML32), ("diff", P.TAP_DIFF), ("msb", P.TAP_MSB)):
        np.testing.assert_array_equal(sess.read_tap(t, n), getattr(orc, k), err_msg=k)
    ref = O.ref_run_local(be, l, 0.375, r, seed, dc, dm, qc, qm, persons, debug_rows=True)
    np.testing.assert_array_equal(sess.row_bits[:n], ref["row_bits"])
    np.testing.assert_array_equal(m, ref["person_match"])
    assert m[0] == 1
    for p in range(3):
        assert sess.last_stats.party(p) == ref["stats"][p]
    np.testing.assert_array_equal(sess.stream_positions(), orc.stream_pos)
