"""Full-scale parity at the BASELINE.json shapes the bench runs (configs[1]
and configs[2]), through the C-ABI on one B200.

At these sizes (up to 1.98e9 lanes) the share-level taps do not fit, so the
check is layered:

* **L1** (per-party additive dots): every query column against a sample of
  256 DB rows (incl. the planted one) plus all 61,504 / 14,880 inner-batch
  pair lanes, captured by `irismpc_gpu_tap_rows`, against the REFERENCE's own
  parse + `kernels::dot_gr_ct_rows` (oracle/_ref, `ref_dots_reshare`) on the
  same payload bytes (the device dealer regenerates those rows bit-exactly).
* **L4** (per-lane opened match bits, `debug_rows`): EVERY lane against the
  plaintext predicate b*(ml - 2hd) > a*ml of tests/oracle.hpp:35-57, computed
  from the plaintext records in C + OpenMP (oracle/plain_bits.c).
* **L5** (opened person bits): against the plaintext OR of each person's lanes;
  the planted person matches.

configs[2] runs the plain limb GEMM over the rotation-pair layout (the S planes
do not fit beside 153.6 GB of DB planes); configs[1] runs the rotation-pair
(Winograd) GEMMs.  Both use the default row-chunk plan.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a B200", allow_module_level=True)

import paper_2405_04463_b200 as P  # noqa: E402
from oracle import pyoracle as O  # noqa: E402

L_BITS, ROT = 12800, 31


def planted_query(sess, S, persons, l=L_BITS):
    """bench.py's query batch: Rng(2) records after the DB; person 0's left eye =
    DB row S/2 rotated by +2 strides with 4 flipped code bits."""
    wl = l // 64
    ncodes = 2 * persons
    codes = torch.empty((ncodes, wl), dtype=torch.int64, device="cuda")
    masks = torch.empty((ncodes, wl), dtype=torch.int64, device="cuda")
    sess.synth_records(2, S, ncodes, 0.9, codes, masks)
    rc_ = torch.empty((1, wl), dtype=torch.int64, device="cuda")
    rm_ = torch.empty((1, wl), dtype=torch.int64, device="cuda")
    sess.synth_records(2, S // 2, 1, 0.9, rc_, rm_)
    c = np.unpackbits(rc_.cpu().numpy().view(np.uint8), bitorder="little")
    m = np.unpackbits(rm_.cpu().numpy().view(np.uint8), bitorder="little")
    by = 2 * (l // 64)
    c, m = np.roll(c, by), np.roll(m, by)
    for f in range(4):
        c[f * (l // 4) + 7] ^= 1
    codes[0] = torch.from_numpy(np.packbits(c, bitorder="little").view(np.int64).copy())
    masks[0] = torch.from_numpy(np.packbits(m, bitorder="little").view(np.int64).copy())
    return codes, masks


def host_records(sess, S, l=L_BITS, chunk=131072):
    """The plaintext DB records [S][l/64] (random_record(l, Rng(2), 0.9)), regenerated on the device."""
    wl = l // 64
    dc = np.empty((S, wl), np.uint64)
    dm = np.empty((S, wl), np.uint64)
    c = torch.empty((chunk, wl), dtype=torch.int64, device="cuda")
    m = torch.empty((chunk, wl), dtype=torch.int64, device="cuda")
    for r0 in range(0, S, chunk):
        n = min(chunk, S - r0)
        sess.synth_records(2, r0, n, 0.9, c[:n], m[:n])
        dc[r0:r0 + n] = c[:n].cpu().numpy().view(np.uint64)
        dm[r0:r0 + n] = m[:n].cpu().numpy().view(np.uint64)
    return dc, dm


def row_payloads(sess, rows, l=L_BITS):
    """The three parties' IRS1 payload bytes of the given DB rows: the device
    dealer regenerates row i from record i of Rng(2) and dealing record i of
    sub_rng(7, 1) (random access into the reference streams)."""
    wl = l // 64
    c = torch.empty((1, wl), dtype=torch.int64, device="cuda")
    m = torch.empty((1, wl), dtype=torch.int64, device="cuda")
    outs = [torch.empty(sess.rec, dtype=torch.uint8, device="cuda") for _ in range(3)]
    pay = [[], [], []]
    for r in rows:
        sess.synth_records(2, int(r), 1, 0.9, c, m)
        sess.deal_payload(7, 1, int(r), c, m, outs)
        for p in range(3):
            pay[p].append(outs[p].cpu().numpy().copy())
    return [np.concatenate(x) for x in pay]


@pytest.mark.parametrize("rows,persons,be", [(100_000, 16, O.SHAMIR), (1_000_000, 32, O.SHAMIR),
                                            (100_000, 16, O.REPLICATED), (1_000_000, 32, O.REPLICATED)],
                         ids=["configs1", "configs2", "configs1-replicated", "configs2-replicated"])
def test_full_scale_parity(rows, persons, be):
    if not O.ref_available():
        pytest.skip("oracle/_ref (the reference built from its sources) is not shipped")
    free, _ = torch.cuda.mem_get_info()
    if rows * 153_600 + (12 << 30) > free:
        pytest.skip("not enough HBM for the DB")
    cfg = P.EngineConfig(backend=be, l=L_BITS, rotations=ROT, debug_rows=True)
    sess = P.Session(cfg, master_seed=7)
    sess.synth_db(rows, rng_seed=2, first=0, mask_density=0.9, deal_seed=7)
    codes, masks = planted_query(sess, rows, persons)
    qpay = [torch.empty(2 * persons * sess.rec, dtype=torch.uint8, device="cuda") for _ in range(3)]
    sess.deal_payload(7, 2, 0, codes, masks, qpay)

    rng = np.random.default_rng(rows)
    sample = np.unique(np.concatenate([rng.choice(rows, 255, replace=False), [rows // 2]])).astype(np.uint64)
    sess.tap_rows(sample)
    match = sess.batch_query(qpay, persons, want_rows=True)
    n = P.lane_count(persons, rows, ROT)
    assert sess.last_stats.lanes == n
    gpu_bits = sess.row_bits[:n]
    dot_hd = sess.read_row_taps(P.TAP_DOT_HD, persons)
    dot_ml = sess.read_row_taps(P.TAP_DOT_ML, persons)
    rp = int(sess.last_stats.rotation_pair_gemm)
    sess.tap_rows([])

    # L1: the reference's own parse + dot kernels on the sampled rows' payload bytes
    db_s = row_payloads(sess, sample)
    qh = [x.cpu().numpy() for x in qpay]
    ref_hd, ref_ml, _, _ = O.ref_dots_reshare(be, L_BITS, ROT, P.seeds_from_master(7), db_s, len(sample), qh,
                                              persons)
    np.testing.assert_array_equal(dot_hd, ref_hd, err_msg=f"L1 hd dots (rotation-pair GEMM: {rp})")
    np.testing.assert_array_equal(dot_ml, ref_ml, err_msg=f"L1 ml dots (rotation-pair GEMM: {rp})")

    # L4 + L5: every lane's opened bit and every person bit vs the plaintext predicate
    dc, dm = host_records(sess, rows)
    qc = codes.cpu().numpy().view(np.uint64)
    qm = masks.cpu().numpy().view(np.uint64)
    _, pers, bad, first = O.plain_batch_bits(L_BITS, ROT, P.MPC_LIFT, 0.375, dc, dm, qc, qm, persons,
                                             expect=gpu_bits, want_bits=False)
    assert bad == 0, f"{bad} of {n} lane bits differ from the plaintext predicate (first at lane {first})"
    np.testing.assert_array_equal(match, pers)
    assert match[0] == 1
    assert gpu_bits[:n - persons * (persons - 1) // 2 * 4 * ROT].sum() > 0


@pytest.mark.parametrize("var", [P.PLAIN_MASK, P.CONST_LIFT, P.NO_LIFT])
def test_full_scale_variants_configs1(var):
    """The other threshold variants at configs[1]'s full shape (32 codes x 31
    rotations x 100k rows, 99.2M lanes): every lane's opened bit (L4) and every person bit (L5)
    against the plaintext predicate of the variant, computed from the plaintext records."""
    rows, persons = 100_000, 16
    cfg = P.EngineConfig(backend=P.SHAMIR, l=L_BITS, rotations=ROT, debug_rows=True, variant=var)
    sess = P.Session(cfg, master_seed=7)
    sess.synth_db(rows, rng_seed=2, first=0, mask_density=0.9, deal_seed=7)
    codes, masks = planted_query(sess, rows, persons)
    qpay = [torch.empty(2 * persons * sess.rec, dtype=torch.uint8, device="cuda") for _ in range(3)]
    sess.deal_payload(7, 2, 0, codes, masks, qpay)
    match = sess.batch_query(qpay, persons, want_rows=True)
    n = P.lane_count(persons, rows, ROT)
    gpu_bits = sess.row_bits[:n]
    dc, dm = host_records(sess, rows)
    qc = codes.cpu().numpy().view(np.uint64)
    qm = masks.cpu().numpy().view(np.uint64)
    _, pers, bad, first = O.plain_batch_bits(L_BITS, ROT, var, 0.375, dc, dm, qc, qm, persons,
                                             expect=gpu_bits, want_bits=False)
    assert bad == 0, f"{bad} of {n} lane bits differ from the plaintext predicate (first at lane {first})"
    np.testing.assert_array_equal(match, pers)
    assert match[0] == 1
