"""GPU parity: the CUDA path through the C-ABI vs the oracle and the golden
vectors of the reference (SURVEY.md §8c levels L1..L5).

L1 per-party additive dots, L2 reshared components, lift/diff/MSB components
(the GPU draws the reference PRF stream layout, so every share through the
MSB is identical), L3 reconstructed distances, L4 per-lane match bits
(debug_rows), L5 opened person bits; plus ledgers and stream positions.
"""
import hashlib
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a B200", allow_module_level=True)

import paper_2405_04463_b200 as P  # noqa: E402
from oracle import pyoracle as O  # noqa: E402

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "ref_vectors.json")))


def _sha(a):
    """oracle/gen_golden.sha: little-endian bytes at the array's ring width."""
    dt = {np.dtype(np.uint16): "<u2", np.dtype(np.uint32): "<u4", np.dtype(np.int64): "<i8"}[a.dtype]
    return hashlib.sha256(np.ascontiguousarray(a).astype(dt).tobytes()).hexdigest()


def _inputs(l, s, persons, seed, membership, planted, density=0.85):
    rng = O.Rng(seed)
    dc, dm = O.records(rng, l, s, density)
    nq = 1 if membership else 2 * persons
    qc, qm = O.records(rng, l, nq, density)
    if planted and s > 0:
        qc[0] = dc[s // 2]
        qm[0] = dm[s // 2]
    return dc, dm, qc, qm


def _gpu(be, l, ratio, r, seed, dc, dm, qc, qm, persons, membership, variant=P.MPC_LIFT):
    cfg = P.EngineConfig(backend=be, l=l, match_ratio=ratio, rotations=r, debug_rows=True, variant=variant)
    m, sess = P.run_batch_local(cfg, qc, qm, dc, dm, seed, persons=persons, membership=membership,
                                want_rows=True, taps=True)
    n = P.lane_count(persons, dc.shape[0], r, membership)
    taps = {k: sess.read_tap(t, n) for k, t in (("dot_hd", P.TAP_DOT_HD), ("dot_ml", P.TAP_DOT_ML),
                                                ("rs_hd", P.TAP_RS_HD), ("rs_ml", P.TAP_RS_ML),
                                                ("ml32", P.TAP_ML32), ("diff", P.TAP_DIFF),
                                                ("msb", P.TAP_MSB))}
    return m, sess, taps, n


@pytest.mark.parametrize("idx", range(len(GOLD["cases"])))
def test_golden_cases(idx):
    c = GOLD["cases"][idx]
    var = c.get("variant", P.MPC_LIFT)
    dc, dm, qc, qm = _inputs(c["l"], c["s"], c["persons"], c["seed"], c["membership"], c["planted"])
    m, sess, taps, n = _gpu(c["backend"], c["l"], c["ratio"], c["rotations"], c["seed"], dc, dm, qc, qm,
                            c["persons"], c["membership"], var)
    assert n == c["lanes"]
    assert [int(x) for x in m] == c["person_match"]                                   # L5
    assert np.packbits(sess.row_bits[:n], bitorder="little").tobytes().hex() == c["row_bits_hex"]  # L4
    assert _sha(taps["dot_hd"]) == c["sha256"]["dot_hd"]                              # L1
    assert _sha(taps["rs_hd"]) == c["sha256"]["rs_hd"]                                # L2
    if P.VARIANT_WIDTHS[var][1]:
        assert _sha(taps["dot_ml"]) == c["sha256"]["dot_ml"]
        assert _sha(taps["rs_ml"]) == c["sha256"]["rs_ml"]
    else:
        assert _sha(taps["dot_ml"].astype(np.int64)) == c["sha256"]["public_ml"]
    st = sess.last_stats
    for p in range(3):
        assert st.party(p) == c["stats"][p]


@pytest.mark.parametrize("be,l,s,persons,r,seed", [
    (O.SHAMIR, 12800, 300, 3, 31, 21),
    (O.REPLICATED, 12800, 300, 3, 31, 22),
    (O.SHAMIR, 12800, 1031, 1, 31, 23),     # s not a multiple of 64/128/1024
    (O.REPLICATED, 256, 2500, 2, 5, 24),
    (O.SHAMIR, 128, 1, 4, 31, 25),          # one DB row
    (O.REPLICATED, 128, 0, 5, 31, 26),      # empty DB, pairs only
])
def test_shares_through_msb_match_oracle(be, l, s, persons, r, seed):
    dc, dm, qc, qm = _inputs(l, s, persons, seed, False, True, 0.9)
    m, sess, taps, n = _gpu(be, l, 0.375, r, seed, dc, dm, qc, qm, persons, False)
    cfg = O.make_config(be, l, 0.375, r, debug_rows=True)
    ref = O.run_local(cfg, seed, dc, dm, qc, qm, persons, want_all=True)
    for k in ("dot_hd", "dot_ml", "rs_hd", "rs_ml", "ml32", "diff", "msb"):
        np.testing.assert_array_equal(taps[k], getattr(ref, k), err_msg=k)
    np.testing.assert_array_equal(sess.row_bits[:n], ref.row_bits)
    np.testing.assert_array_equal(m, ref.person_match)
    np.testing.assert_array_equal(sess.read_tap(P.TAP_AGG, persons), ref.agg)  # OR-tree shares
    np.testing.assert_array_equal(sess.stream_positions(), ref.stream_pos)
    # L3: reconstructed distances equal the plaintext ones
    rec_ml = taps["rs_ml"].astype(np.uint32).sum(0) & 0xFFFF
    rec_hd = taps["rs_hd"].astype(np.uint32).sum(0) & 0xFFFF
    np.testing.assert_array_equal(rec_ml, ref.rs_ml.astype(np.uint32).sum(0) & 0xFFFF)
    np.testing.assert_array_equal(rec_hd, ref.rs_hd.astype(np.uint32).sum(0) & 0xFFFF)


@pytest.mark.parametrize("var", [P.PLAIN_MASK, P.CONST_LIFT, P.NO_LIFT])
@pytest.mark.parametrize("be,l,s,persons,r,seed", [
    (O.SHAMIR, 12800, 300, 3, 31, 41),
    (O.REPLICATED, 12800, 260, 2, 31, 42),
    (O.SHAMIR, 256, 1031, 2, 5, 43),
    (O.REPLICATED, 128, 1, 4, 31, 44),      # one DB row
    (O.SHAMIR, 128, 0, 3, 3, 45),           # empty DB, pairs only
])
def test_variant_shares_through_msb_match_oracle(var, be, l, s, persons, r, seed):
    """f1: plain-mask / const-lift / no-lift, every share through the MSB."""
    dc, dm, qc, qm = _inputs(l, s, persons, seed, False, True, 0.9)
    m, sess, taps, n = _gpu(be, l, 0.375, r, seed, dc, dm, qc, qm, persons, False, var)
    ref = O.run_local(O.make_config(be, l, 0.375, r, debug_rows=True, variant=var), seed, dc, dm, qc, qm,
                      persons, want_all=True)
    for k in ("dot_hd", "rs_hd", "rs_ml", "ml32", "diff", "msb"):
        np.testing.assert_array_equal(taps[k], getattr(ref, k), err_msg=k)
    if P.VARIANT_WIDTHS[var][1]:
        np.testing.assert_array_equal(taps["dot_ml"], ref.dot_ml)
    else:
        np.testing.assert_array_equal(taps["dot_ml"], ref.public_ml)
    np.testing.assert_array_equal(sess.row_bits[:n], ref.row_bits)
    np.testing.assert_array_equal(m, ref.person_match)
    np.testing.assert_array_equal(sess.read_tap(P.TAP_AGG, persons), ref.agg)
    np.testing.assert_array_equal(sess.stream_positions(), ref.stream_pos)
    st = sess.last_stats
    for p in range(3):
        assert st.party(p) == ref.stats[p]


@pytest.mark.parametrize("var", [P.PLAIN_MASK, P.CONST_LIFT, P.NO_LIFT])
@pytest.mark.parametrize("be", [O.SHAMIR, O.REPLICATED])
def test_variant_membership(var, be):
    l, s = 64, 300
    dc, dm, qc, qm = _inputs(l, s, 1, 78, True, True, 0.8)
    cfg = P.EngineConfig(backend=be, l=l, rotations=1, debug_rows=True, variant=var)
    m, sess = P.run_batch_local(cfg, qc, qm, dc, dm, 78, membership=True, want_rows=True)
    ref = O.run_local(O.make_config(be, l, 0.375, 1, True, variant=var), 78, dc, dm, qc, qm, 1, membership=True)
    assert m[0] == ref.person_match[0] == 1
    np.testing.assert_array_equal(sess.row_bits[:s], ref.row_bits)


@pytest.mark.parametrize("var", [P.PLAIN_MASK, P.CONST_LIFT, P.NO_LIFT])
@pytest.mark.parametrize("be", [O.SHAMIR, O.REPLICATED])
def test_variant_device_dealer(var, be):
    l, n = 256, 7
    sess = P.Session(P.EngineConfig(backend=be, l=l, variant=var), master_seed=1)
    rng = O.Rng(5)
    oc, om = O.records(rng, l, n, 0.9)
    codes = torch.from_numpy(oc.view(np.int64)).cuda()
    masks = torch.from_numpy(om.view(np.int64)).cuda()
    outs = [torch.empty(n * sess.rec, dtype=torch.uint8, device="cuda") for _ in range(3)]
    sess.deal_payload(7, 1, 0, codes, masks, outs)
    ref = O.deal(be, l, oc, om, O.Rng(sub=(7, 1)), variant=var)
    for a, b in zip(outs, ref):
        np.testing.assert_array_equal(a.cpu().numpy(), b)


@pytest.mark.parametrize("var", [P.MPC_LIFT, P.NO_LIFT])
def test_accumulator_wraparound_all_ones_shares(var):
    """Replicated all-0xFF payloads are consistent shares whose limb products
    overflow the s32 TMEM accumulators (K = 2l = 25600: 2 x 25600 x 255^2 > 2^31);
    the dots are only needed mod 2^K, so the wrap must be exact."""
    l, s, persons, r, seed = 12800, 256, 1, 31, 61
    rec = O.record_bytes(O.REPLICATED, l, var)
    db = [np.full(s * rec, 0xFF, np.uint8) for _ in range(3)]
    q = [np.full(2 * persons * rec, 0xFF, np.uint8) for _ in range(3)]
    seeds = O.party_seeds(seed)
    cfg = P.EngineConfig(backend=O.REPLICATED, l=l, rotations=r, debug_rows=True, variant=var)
    sess = P.Session(cfg, seeds=seeds)
    sess.load_db(db, s)
    sess.enable_taps(True)
    m = sess.batch_query(q, persons, want_rows=True)
    n = P.lane_count(persons, s, r)
    ref = O.query(O.make_config(O.REPLICATED, l, 0.375, r, debug_rows=True, variant=var), seeds, db, s, q,
                  persons, want_all=True)
    np.testing.assert_array_equal(sess.read_tap(P.TAP_DOT_HD, n), ref.dot_hd)
    np.testing.assert_array_equal(sess.read_tap(P.TAP_DOT_ML, n), ref.dot_ml)
    np.testing.assert_array_equal(sess.row_bits[:n], ref.row_bits)
    np.testing.assert_array_equal(m, ref.person_match)


@pytest.mark.parametrize("be", [O.SHAMIR, O.REPLICATED])
def test_membership_and_planted(be):
    l, s = 64, 200
    dc, dm, qc, qm = _inputs(l, s, 1, 77, True, True, 0.8)
    cfg = P.EngineConfig(backend=be, l=l, rotations=1, debug_rows=True)
    m, sess = P.run_batch_local(cfg, qc, qm, dc, dm, 77, membership=True, want_rows=True)
    ref = O.run_local(O.make_config(be, l, 0.375, 1, True), 77, dc, dm, qc, qm, 1, membership=True)
    assert m[0] == ref.person_match[0] == 1
    np.testing.assert_array_equal(sess.row_bits[:s], ref.row_bits)


@pytest.mark.parametrize("be", [O.SHAMIR, O.REPLICATED])
def test_device_dealer_matches_reference_dealer(be):
    l, n = 12800, 5
    sess = P.Session(P.EngineConfig(backend=be, l=l), master_seed=1)
    wl = (l + 63) // 64
    codes = torch.empty((n, wl), dtype=torch.int64, device="cuda")
    masks = torch.empty((n, wl), dtype=torch.int64, device="cuda")
    sess.synth_records(2, 3, n, 0.9, codes, masks)
    rng = O.Rng(2)
    O.records(rng, l, 3, 0.9)  # skip 3 records
    oc, om = O.records(rng, l, n, 0.9)
    np.testing.assert_array_equal(codes.cpu().numpy().view(np.uint64), oc)
    np.testing.assert_array_equal(masks.cpu().numpy().view(np.uint64), om)
    outs = [torch.empty(n * sess.rec, dtype=torch.uint8, device="cuda") for _ in range(3)]
    sess.deal_payload(7, 1, 0, codes, masks, outs)
    ref = O.deal(be, l, oc, om, O.Rng(sub=(7, 1)))
    for a, b in zip(outs, ref):
        np.testing.assert_array_equal(a.cpu().numpy(), b)


def test_host_and_device_payload_paths_agree():
    l, s, persons, seed = 12800, 64, 2, 31
    dc, dm, qc, qm = _inputs(l, s, persons, seed, False, True, 0.9)
    db = O.deal(O.SHAMIR, l, dc, dm, O.Rng(sub=(seed, 1)))
    q = O.deal(O.SHAMIR, l, qc, qm, O.Rng(sub=(seed, 2)))
    cfg = P.EngineConfig(backend=P.SHAMIR, l=l)
    a = P.Session(cfg, master_seed=seed)
    a.load_db(db, s)
    ma = a.batch_query(q, persons)
    b = P.Session(cfg, master_seed=seed)
    b.load_db([torch.from_numpy(x).cuda() for x in db], s)
    mb = b.batch_query([torch.from_numpy(x).cuda() for x in q], persons)
    ref = O.run_local(O.make_config(O.SHAMIR, l), seed, dc, dm, qc, qm, persons)
    np.testing.assert_array_equal(ma, ref.person_match)
    np.testing.assert_array_equal(mb, ref.person_match)
    # persistent context: second query continues the streams like the reference CLI
    np.testing.assert_array_equal(a.stream_positions(), ref.stream_pos)
    ma2 = a.batch_query(q, persons)
    ref2 = O.query(O.make_config(O.SHAMIR, l), O.party_seeds(seed), db, s, q, persons,
                   stream_start=ref.stream_pos)
    np.testing.assert_array_equal(ma2, ref2.person_match)
    np.testing.assert_array_equal(a.stream_positions(), ref2.stream_pos)


def test_payload_errors_map_to_reference_exceptions():
    l = 64
    sess = P.Session(P.EngineConfig(backend=P.REPLICATED, l=l, rotations=1), master_seed=3)
    rec = sess.rec
    with pytest.raises(P.ConfigError):          # "db payload size mismatch"
        sess.load_db([np.zeros(rec * 2 + 1, np.uint8)] * 3, 2)
    with pytest.raises(P.InconsistentShareError):  # replication cross-check
        sess.load_db([np.random.default_rng(0).integers(0, 255, rec * 2, dtype=np.uint8) for _ in range(3)], 2)
    dc, dm, qc, qm = _inputs(l, 4, 1, 5, False, False)
    db = O.deal(O.REPLICATED, l, dc, dm, O.Rng(sub=(5, 1)))
    sess.load_db(db, 4)
    with pytest.raises(P.ConfigError):          # "batch query expects 2 codes per person"
        sess.batch_query([np.zeros(rec, np.uint8)] * 3, 1)


@pytest.mark.parametrize("be,var", [(O.SHAMIR, P.MPC_LIFT), (O.REPLICATED, P.PLAIN_MASK), (O.SHAMIR, P.NO_LIFT)])
def test_configs2_batch_shape_32_persons(be, var):
    """configs[2]'s batch shape: 64 codes (32 persons) x 31 rotations = 1984 columns
    (8 column tiles of 256) and 61 504 inner-batch pair lanes, at a DB size the
    oracle finishes quickly; every lane bit and person bit vs the oracle.  Persons
    5 and 20 carry planted DB rows; person 11's right eye is person 3's left eye."""
    l, s, persons, r, seed = 2048, 300, 32, 31, 51
    dc, dm, qc, qm = _inputs(l, s, persons, seed, False, False, 0.9)
    qc[10], qm[10] = dc[17], dm[17]
    qc[41], qm[41] = dc[250], dm[250]
    qc[23], qm[23] = qc[6], qm[6]
    cfg = P.EngineConfig(backend=be, l=l, rotations=r, debug_rows=True, variant=var)
    m, sess = P.run_batch_local(cfg, qc, qm, dc, dm, seed, persons=persons, want_rows=True)
    ref = O.run_local(O.make_config(be, l, 0.375, r, debug_rows=True, variant=var), seed, dc, dm, qc, qm, persons)
    n = P.lane_count(persons, s, r)
    assert n == 64 * r * s + 61_504
    np.testing.assert_array_equal(sess.row_bits[:n], ref.row_bits)
    np.testing.assert_array_equal(m, ref.person_match)
    assert m[5] == 1 and m[20] == 1 and m[11] == 1 and m[3] == 1
    np.testing.assert_array_equal(sess.stream_positions(), ref.stream_pos)


def test_sharded_db_matches_single_gpu():
    """Two shards on one GPU (rows split), partial shares + MPC OR + open."""
    l, s, persons, seed = 12800, 700, 2, 41
    dc, dm, qc, qm = _inputs(l, s, persons, seed, False, True, 0.9)
    db = O.deal(O.SHAMIR, l, dc, dm, O.Rng(sub=(seed, 1)))
    q = O.deal(O.SHAMIR, l, qc, qm, O.Rng(sub=(seed, 2)))
    rec = O.record_bytes(O.SHAMIR, l)
    cfg = P.EngineConfig(backend=P.SHAMIR, l=l)
    split = 333
    qd = [torch.from_numpy(x).cuda() for x in q]
    parts = torch.zeros((2, 3, persons), dtype=torch.uint8, device="cuda")
    sessions = []
    for rank, (r0, r1) in enumerate([(0, split), (split, s)]):
        sh = P.Session(cfg, master_seed=seed, shard_rank=rank, db_rows_total=s, db_row_offset=r0)
        sh.load_db([x[r0 * rec:r1 * rec] for x in db], r1 - r0)
        sh.batch_query_partial(qd, persons, parts[rank])
        sessions.append(sh)
    m = sessions[0].or_open(parts, 2, persons)
    ref = O.run_local(O.make_config(O.SHAMIR, l), seed, dc, dm, qc, qm, persons)
    np.testing.assert_array_equal(m, ref.person_match)
    assert m[0] == 1


def test_full_size_synthetic_planted_match():
    """Size-independent property at the headline scale: a planted rotated
    near-copy of DB row s/2 is found; a DB of fresh random rows is not."""
    l, s, persons = 12800, 100_000, 16
    cfg = P.EngineConfig(backend=P.SHAMIR, l=l)
    sess = P.Session(cfg, master_seed=7)
    sess.synth_db(s, rng_seed=2, first=0, mask_density=0.9, deal_seed=7)
    wl = l // 64
    codes = torch.empty((2 * persons, wl), dtype=torch.int64, device="cuda")
    masks = torch.empty((2 * persons, wl), dtype=torch.int64, device="cuda")
    sess.synth_records(2, s, 2 * persons, 0.9, codes, masks)
    row = torch.empty((1, wl), dtype=torch.int64, device="cuda")
    rowm = torch.empty((1, wl), dtype=torch.int64, device="cuda")
    sess.synth_records(2, s // 2, 1, 0.9, row, rowm)
    c = np.unpackbits(row.cpu().numpy().view(np.uint8), bitorder="little")
    mk = np.unpackbits(rowm.cpu().numpy().view(np.uint8), bitorder="little")
    by = 2 * (l // 64)
    c, mk = np.roll(c, by), np.roll(mk, by)
    for f in range(4):
        c[f * (l // 4) + 7] ^= 1
    codes[0] = torch.from_numpy(np.packbits(c, bitorder="little").view(np.int64).copy())
    masks[0] = torch.from_numpy(np.packbits(mk, bitorder="little").view(np.int64).copy())
    outs = [torch.empty(2 * persons * sess.rec, dtype=torch.uint8, device="cuda") for _ in range(3)]
    sess.deal_payload(7, 2, 0, codes, masks, outs)
    m = sess.batch_query(outs, persons)
    assert m[0] == 1 and m[1:].sum() == 0
    assert sess.last_stats.lanes == P.lane_count(persons, s, 31)


@pytest.mark.parametrize("chunk_lanes,thr_lanes", [("1000000000", "7000"), ("60000", "1000000000"),
                                                   ("30000", "7000")])
def test_threshold_job_splits(chunk_lanes, thr_lanes):
    """DB lanes run in row chunks (GEMM || threshold on two streams) and each
    chunk's threshold in column jobs; neither split may change any output."""
    import subprocess, sys, textwrap
    code = textwrap.dedent("""
        import sys, numpy as np
        sys.path.insert(0, '.')
        import paper_2405_04463_b200 as P
        from oracle import pyoracle as O
        l, s, persons, seed = 256, 3000, 3, 61
        rng = O.Rng(seed)
        dc, dm = O.records(rng, l, s, 0.9)
        qc, qm = O.records(rng, l, 2 * persons, 0.9)
        qc[2], qm[2] = dc[17], dm[17]
        cfg = P.EngineConfig(backend=P.SHAMIR, l=l, rotations=5, debug_rows=True)
        m, sess = P.run_batch_local(cfg, qc, qm, dc, dm, seed, persons=persons, want_rows=True)
        ref = O.run_local(O.make_config(O.SHAMIR, l, 0.375, 5, True), seed, dc, dm, qc, qm, persons)
        n = P.lane_count(persons, s, 5)
        assert (m == ref.person_match).all(), (m, ref.person_match)
        assert (sess.row_bits[:n] == ref.row_bits).all()
        print("ok", m)
    """)
    import os
    env = dict(os.environ, IRISMPC_THR_LANES=thr_lanes, IRISMPC_CHUNK_LANES=chunk_lanes)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.parametrize("be,var", [(O.SHAMIR, P.MPC_LIFT), (O.REPLICATED, P.CONST_LIFT), (O.SHAMIR, P.PLAIN_MASK)])
def test_persistent_session_varying_query_shapes(be, var):
    """One context, queries of changing shape (persons 3 -> membership -> 9 -> 1 -> 5): buffers
    are resized between calls and the PRF streams keep advancing like a CLI PartyCtx; every
    query's row bits and person bits equal the oracle's started at the carried positions."""
    l, s, r, seed = 256, 700, 5, 91
    rng = O.Rng(seed)
    dc, dm = O.records(rng, l, s, 0.9)
    db = O.deal(be, l, dc, dm, O.Rng(sub=(seed, 1)), variant=var)
    seeds = O.party_seeds(seed)
    cfg = P.EngineConfig(backend=be, l=l, rotations=r, debug_rows=True, variant=var)
    sess = P.Session(cfg, seeds=seeds)
    sess.load_db(db, s)
    pos = np.zeros(3, np.uint64)
    for qi, (persons, memb) in enumerate([(3, False), (1, True), (9, False), (1, False), (5, False)]):
        nq = 1 if memb else 2 * persons
        qc, qm = O.records(rng, l, nq, 0.9)
        qc[0], qm[0] = dc[(37 * qi) % s], dm[(37 * qi) % s]
        q = O.deal(be, l, qc, qm, O.Rng(sub=(seed, 10 + qi)), variant=var)
        rr = 1 if memb else r
        ref = O.query(O.make_config(be, l, 0.375, rr, debug_rows=True, variant=var), seeds, db, s, q,
                      persons, membership=memb, stream_start=pos)
        if memb:
            m = np.array([sess.membership(q, want_rows=True)], np.uint8)
            n = s
        else:
            m = sess.batch_query(q, persons, want_rows=True)
            n = P.lane_count(persons, s, r)
        np.testing.assert_array_equal(m, ref.person_match, err_msg=f"query {qi}")
        np.testing.assert_array_equal(sess.row_bits[:n], ref.row_bits, err_msg=f"query {qi}")
        np.testing.assert_array_equal(sess.stream_positions(), ref.stream_pos, err_msg=f"query {qi}")
        assert m[0] == 1
        pos = ref.stream_pos


@pytest.mark.parametrize("mode", ["1", "layout", "0", "chunked", "conv"])
@pytest.mark.parametrize("be,var,l", [(O.SHAMIR, P.MPC_LIFT, 1024), (O.REPLICATED, P.NO_LIFT, 512),
                                      (O.SHAMIR, P.PLAIN_MASK, 1024)])
def test_rotation_pair_gemm_modes(mode, be, var, l):
    """The rotation-pair (Winograd F(2,2)) GEMMs, the RP plane layout without
    them (the large-DB fallback) and the natural layout: per-party dots (L1),
    row bits and person bits identical to the oracle in every mode."""
    import subprocess, sys, textwrap
    code = textwrap.dedent(f"""
        import sys, numpy as np
        sys.path.insert(0, '.')
        import paper_2405_04463_b200 as P
        from oracle import pyoracle as O
        be, var, l, s, persons, seed, r = {be}, {var}, {l}, 700, 2, 23, 31
        rng = O.Rng(seed)
        dc, dm = O.records(rng, l, s, 0.9)
        qc, qm = O.records(rng, l, 2 * persons, 0.9)
        qc[1], qm[1] = dc[300], dm[300]
        cfg = P.EngineConfig(backend=be, l=l, rotations=r, debug_rows=True, variant=var)
        m, sess = P.run_batch_local(cfg, qc, qm, dc, dm, seed, persons=persons, want_rows=True, taps=True)
        ref = O.run_local(O.make_config(be, l, 0.375, r, True, variant=var), seed, dc, dm, qc, qm, persons,
                          want_all=True)
        n = P.lane_count(persons, s, r)
        assert (m == ref.person_match).all(), (m, ref.person_match)
        assert (sess.row_bits[:n] == ref.row_bits).all()
        np.testing.assert_array_equal(sess.read_tap(P.TAP_DOT_HD, n), ref.dot_hd, err_msg="L1 hd dots")
        if var != P.PLAIN_MASK:
            np.testing.assert_array_equal(sess.read_tap(P.TAP_DOT_ML, n), ref.dot_ml, err_msg="L1 ml dots")
        np.testing.assert_array_equal(sess.stream_positions(), ref.stream_pos)
        rp = int(sess.last_stats.rotation_pair_gemm)
        assert rp == (1 if {mode!r} in ("1", "chunked", "conv") else 0), rp
        print("ok", m, rp)
    """)
    import os
    env = dict(os.environ, IRISMPC_RP=mode, IRISMPC_RP_FORCE="1")
    if mode == "chunked":  # S planes built per row chunk (large-DB path), three row chunks
        env.update(IRISMPC_RP="1", IRISMPC_RP_CHUNKED="force", IRISMPC_CHUNK_LANES="8000")
    if mode == "conv":  # S = E + O formed in the GEMM's shared memory, three row chunks
        env.update(IRISMPC_RP="1", IRISMPC_RP_CHUNKED="conv_force", IRISMPC_CHUNK_LANES="8000")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.parametrize("be,l,r,persons,s", [(O.SHAMIR, 1024, 3, 1, 300), (O.REPLICATED, 512, 5, 3, 257),
                                              (O.SHAMIR, 2048, 31, 1, 1)])
def test_rotation_pair_gemm_shapes(be, l, r, persons, s, monkeypatch):
    """Rotation-pair GEMMs at other rotation counts (an odd number of pairs' last
    rotation dropped), one person, a one-row DB: shares through the MSB and the
    opened bits identical to the oracle.  (These batches are too narrow for the
    rotation-pair GEMMs to pay, so IRISMPC_RP_FORCE selects them.)"""
    monkeypatch.setenv("IRISMPC_RP_FORCE", "1")
    dc, dm, qc, qm = _inputs(l, s, persons, 77, False, True, 0.9)
    m, sess, taps, n = _gpu(be, l, 0.375, r, 77, dc, dm, qc, qm, persons, False)
    ref = O.run_local(O.make_config(be, l, 0.375, r, debug_rows=True), 77, dc, dm, qc, qm, persons, want_all=True)
    for k in ("dot_hd", "dot_ml", "rs_hd", "rs_ml", "diff", "msb"):
        np.testing.assert_array_equal(taps[k], getattr(ref, k), err_msg=k)
    np.testing.assert_array_equal(sess.row_bits[:n], ref.row_bits)
    np.testing.assert_array_equal(m, ref.person_match)
    assert sess.last_stats.rotation_pair_gemm == 1


@pytest.mark.parametrize("be,var,s", [(O.SHAMIR, P.MPC_LIFT, 3000), (O.REPLICATED, P.PLAIN_MASK, 700),
                                      (O.SHAMIR, P.NO_LIFT, 1500)])
def test_streaming_queries_match_synchronous(be, var, s):
    """irismpc_gpu_batch_query_submit / _wait: five queries with two in flight
    (the GEMM stream runs into the next query while the threshold finishes the
    previous one) give the oracle's person bits at the carried stream positions,
    and the final positions equal the synchronous sequence's."""
    l, r, seed, persons = 256, 5, 17, 3
    rng = O.Rng(seed)
    dc, dm = O.records(rng, l, s, 0.9)
    db = O.deal(be, l, dc, dm, O.Rng(sub=(seed, 1)), variant=var)
    seeds = O.party_seeds(seed)
    cfg = P.EngineConfig(backend=be, l=l, rotations=r, variant=var)
    qs = []
    for i in range(5):
        qc, qm = O.records(rng, l, 2 * persons, 0.9)
        qc[(2 * i) % (2 * persons)], qm[(2 * i) % (2 * persons)] = dc[(53 * i) % s], dm[(53 * i) % s]
        qs.append(O.deal(be, l, qc, qm, O.Rng(sub=(seed, 10 + i)), variant=var))
    sess = P.Session(cfg, seeds=seeds)
    sess.load_db(db, s)
    qd = [[torch.from_numpy(x).cuda() for x in q] for q in qs]
    tickets, got = [], []
    for i, q in enumerate(qd):
        tickets.append(sess.batch_query_submit(q, persons))
        if i >= 1:
            got.append(sess.batch_query_wait(tickets[i - 1]))
    got.append(sess.batch_query_wait(tickets[-1]))
    pos = np.zeros(3, np.uint64)
    for i, q in enumerate(qs):
        ref = O.query(O.make_config(be, l, 0.375, r, variant=var), seeds, db, s, q, persons, stream_start=pos)
        np.testing.assert_array_equal(got[i], ref.person_match, err_msg=f"query {i}")
        assert got[i].any()
        pos = ref.stream_pos
    np.testing.assert_array_equal(sess.stream_positions(), pos)
    np.testing.assert_array_equal(sess.read_tap(P.TAP_AGG, persons), ref.agg)  # the last query's OR tree


def test_streaming_queries_multi_chunk():
    """The streaming path with several row chunks per query (dot-buffer halves
    alternate across the query boundary), in a fresh process with small chunks."""
    import os
    import subprocess
    import sys
    code = (
        "import sys; sys.path.insert(0, '.'); sys.path.insert(0, 'tests');"
        "import test_gpu_parity as T; T.test_streaming_queries_match_synchronous(1, 1, 3000);"
        "T.test_streaming_queries_match_synchronous(0, 3, 1500); print('ok')")
    env = dict(os.environ, IRISMPC_CHUNK_LANES="20000")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


@pytest.mark.parametrize("kernels", ["tile", "lm"])
def test_threshold_kernel_variants_share_exact(kernels):
    """Both reshare / inject implementations (the lane-major kernels a batch query
    uses beside the GEMM, the 504-lane tile kernels of the comparison-only path)
    forced on batch queries: every share through the MSB equals the oracle's, for
    all four variants and both backends (fresh process per variant: the selection
    is read once)."""
    import os
    import subprocess
    import sys
    code = (
        "import sys; sys.path.insert(0, '.'); sys.path.insert(0, 'tests');"
        "import test_gpu_parity as T;"
        "T.test_shares_through_msb_match_oracle(1, 12800, 1031, 1, 31, 23);"
        "T.test_shares_through_msb_match_oracle(0, 256, 2500, 2, 5, 24);"
        "[T.test_variant_shares_through_msb_match_oracle(v, 1, 256, 1031, 2, 5, 43) for v in (0, 2, 3)];"
        "[T.test_variant_shares_through_msb_match_oracle(v, 0, 128, 1, 4, 31, 44) for v in (0, 2, 3)];"
        "print('ok')")
    env = dict(os.environ, IRISMPC_THR_KERNELS=kernels, IRISMPC_CHUNK_LANES="30000")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


@pytest.mark.parametrize("persons,rp", [(4, 0), (8, 1), (16, 1)])
def test_rotation_pair_gemm_chosen_by_tile_cost(persons, rp):
    """The rotation-pair GEMMs run when their padded column tiles cost less than
    the plain GEMM's (3 ceil(16 codes'/256) < 2 ceil(31 codes/256)): not for a
    batch of 8 codes (128 pair columns half-fill a tile), yes from 16 codes."""
    l, s, r, seed = 1024, 300, 31, 5
    dc, dm, qc, qm = _inputs(l, s, persons, seed, False, True, 0.9)
    m, sess, taps, n = _gpu(O.SHAMIR, l, 0.375, r, seed, dc, dm, qc, qm, persons, False)
    assert sess.last_stats.rotation_pair_gemm == rp
    ref = O.run_local(O.make_config(O.SHAMIR, l, 0.375, r, debug_rows=True), seed, dc, dm, qc, qm, persons)
    np.testing.assert_array_equal(m, ref.person_match)
    np.testing.assert_array_equal(sess.row_bits[:n], ref.row_bits)


@pytest.mark.parametrize("persons,rp", [(64, "1"), (128, "1"), (128, "0")])
def test_wide_batch_shares_match_oracle(persons, rp):
    """Wide batches (128 / 256 codes: 16 / 31 column tiles, more than whole cluster
    groups fit, so the persistent GEMM walks its tiles ungrouped), with and without
    the rotation-pair GEMMs: per-party dots (L1), row bits, person bits and the
    OR-tree shares equal the oracle's."""
    import subprocess, sys, textwrap
    code = textwrap.dedent(f"""
        import sys, numpy as np
        sys.path.insert(0, '.')
        import paper_2405_04463_b200 as P
        from oracle import pyoracle as O
        be, l, s, persons, seed, r = O.SHAMIR, 512, 200, {persons}, 29, 31
        rng = O.Rng(seed)
        dc, dm = O.records(rng, l, s, 0.9)
        qc, qm = O.records(rng, l, 2 * persons, 0.9)
        qc[2 * persons - 1], qm[2 * persons - 1] = dc[199], dm[199]
        cfg = P.EngineConfig(backend=be, l=l, rotations=r, debug_rows=True)
        m, sess = P.run_batch_local(cfg, qc, qm, dc, dm, seed, persons=persons, want_rows=True, taps=True)
        ref = O.run_local(O.make_config(be, l, 0.375, r, True), seed, dc, dm, qc, qm, persons, want_all=True)
        n = P.lane_count(persons, s, r)
        assert (m == ref.person_match).all() and m[-1] == 1 and m.sum() < persons // 2
        assert (sess.row_bits[:n] == ref.row_bits).all()
        np.testing.assert_array_equal(sess.read_tap(P.TAP_DOT_HD, n), ref.dot_hd, err_msg="L1 hd dots")
        np.testing.assert_array_equal(sess.read_tap(P.TAP_DOT_ML, n), ref.dot_ml, err_msg="L1 ml dots")
        np.testing.assert_array_equal(sess.read_tap(P.TAP_AGG, persons), ref.agg)
        print("ok", int(sess.last_stats.rotation_pair_gemm))
    """)
    import os
    env = dict(os.environ, IRISMPC_RP=rp)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


def test_sharded_shares_are_shard_count_invariant():
    """lane and PRF indices are global, so each shard's reshared
    components, comparison inputs and MSB components at its lanes equal the
    single-context reference's, share for share (two shards, rows split)."""
    l, s, persons, seed, r = 256, 700, 2, 43, 5
    dc, dm, qc, qm = _inputs(l, s, persons, seed, False, True, 0.9)
    db = O.deal(O.SHAMIR, l, dc, dm, O.Rng(sub=(seed, 1)))
    q = O.deal(O.SHAMIR, l, qc, qm, O.Rng(sub=(seed, 2)))
    rec = O.record_bytes(O.SHAMIR, l)
    cfg = P.EngineConfig(backend=P.SHAMIR, l=l, rotations=r)
    ref = O.run_local(O.make_config(O.SHAMIR, l, 0.375, r), seed, dc, dm, qc, qm, persons, want_all=True)
    n = P.lane_count(persons, s, r)
    ncols = 2 * persons * r
    qd = [torch.from_numpy(x).cuda() for x in q]
    parts = torch.zeros((2, 3, persons), dtype=torch.uint8, device="cuda")
    for rank, (r0, r1) in enumerate([(0, 333), (333, s)]):
        sh = P.Session(cfg, master_seed=seed, shard_rank=rank, db_rows_total=s, db_row_offset=r0)
        sh.load_db([x[r0 * rec:r1 * rec] for x in db], r1 - r0)
        sh.enable_taps(True)
        sh.batch_query_partial(qd, persons, parts[rank])
        lanes = np.concatenate([col * s + np.arange(r0, r1) for col in range(ncols)])
        if rank == 0:  # the inner-batch pair lanes run on shard 0
            lanes = np.concatenate([lanes, np.arange(ncols * s, n)])
        # (the full L1 dot taps are single-context only; the reshared components already pin them)
        for k, t in (("rs_hd", P.TAP_RS_HD), ("rs_ml", P.TAP_RS_ML), ("diff", P.TAP_DIFF), ("msb", P.TAP_MSB)):
            got = sh.read_tap(t, n)
            np.testing.assert_array_equal(got[:, lanes], getattr(ref, k)[:, lanes], err_msg=f"{k} shard {rank}")
