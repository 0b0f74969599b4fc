"""The comparison phase alone on the B200 (irismpc_gpu_comparison_only /
irismpc_gpu_or_tree_only) vs the reference's party_comparison_only /
party_or_tree_only (src/engine.cpp:448-532, run through run_comparison_local /
run_or_tree_local of oracle/_ref): every lane's opened MSB bit equals the
plaintext predicate, the opened OR equals the reference's, and each party's
ledger (lift, ot, msb, or_tree bytes) equals the reference's CommLedger."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a B200", allow_module_level=True)

import paper_2405_04463_b200 as P  # noqa: E402
from oracle import pyoracle as O  # noqa: E402


def _predicate(dots, mls, variant, ratio=0.375):
    if variant == P.PLAIN_MASK:
        return (dots > np.ceil((1 - 2 * ratio) * mls).astype(np.int64)).astype(np.uint8)
    a = O.lib().orc_match_a(ratio)
    return ((1 << 16) * dots > a * mls).astype(np.uint8)


def _payloads(dots, mls, variant, rng):
    kh, km, _ = P.VARIANT_WIDTHS[variant]
    hp = P.share_lane_values(dots, kh, rng)
    mp = P.share_lane_values(mls, km, rng) if km else [mls.astype("<u8").view(np.uint8)] * 3
    return hp, mp


@pytest.mark.parametrize("var", [P.PLAIN_MASK, P.MPC_LIFT, P.CONST_LIFT, P.NO_LIFT])
@pytest.mark.parametrize("n", [1, 1000, 100_000])
def test_comparison_only_matches_reference(var, n):
    dots, mls = O.synth_lanes(n, 12800, 50 + var)
    rng = np.random.default_rng(n + var)
    hp, mp = _payloads(dots, mls, var, rng)
    sess = P.Session(P.EngineConfig(backend=P.REPLICATED, l=12800, rotations=1, variant=var), master_seed=5000)
    opened, bits = sess.comparison_only(hp, mp, n, with_or_tree=True, want_bits=True)
    want = _predicate(dots, mls, var)
    np.testing.assert_array_equal(bits, want)
    assert opened == int(want.any())
    st = sess.last_stats
    if O.ref_available():
        ref = O.ref_comparison_local(var, dots, mls, True, 5000)
        assert ref["opened"] == opened
        for p in range(3):
            led = ref["ledger"][p]
            assert st.lift_bytes[p] == led["lift"] + led["ot"]
            assert st.msb_bytes[p] == led["msb"]
            assert st.or_tree_bytes[p] == led["or_tree"]


def test_comparison_only_multi_job_and_planted_bit():
    """more than 2^24 lanes (two threshold jobs); one lane above the threshold"""
    n = (1 << 24) + 4097
    var = P.MPC_LIFT
    mls = np.full(n, 1000, np.int64)
    dots = np.full(n, -1000, np.int64)
    dots[n - 3] = 1000
    rng = np.random.default_rng(3)
    hp, mp = _payloads(dots, mls, var, rng)
    sess = P.Session(P.EngineConfig(backend=P.REPLICATED, l=12800, rotations=1, variant=var), master_seed=1)
    opened, bits = sess.comparison_only(hp, mp, n, with_or_tree=True, want_bits=True)
    assert opened == 1
    assert bits.sum() == 1 and bits[n - 3] == 1
    opened, _ = sess.comparison_only(hp, mp, n, with_or_tree=False)
    assert opened is None


@pytest.mark.parametrize("n,planted", [(100_000, 12345), (100_000, None), (70, 69), (3_000_000, 2_999_999)])
def test_or_tree_only_matches_reference(n, planted):
    bits = np.zeros(n, np.uint8)
    if planted is not None:
        bits[planted] = 1
    sess = P.Session(P.EngineConfig(backend=P.REPLICATED, l=12800, rotations=1), master_seed=5001)
    opened = sess.or_tree_only(P.share_bit_words(bits, np.random.default_rng(n)), n)
    assert opened == int(bits.any())
    if O.ref_available():
        ref = O.ref_or_tree_local(bits, 5001)
        assert ref["opened"] == opened
        assert [sess.last_stats.or_tree_bytes[p] for p in range(3)] == ref["or_bytes"]


def test_comparison_payload_errors():
    sess = P.Session(P.EngineConfig(backend=P.REPLICATED, l=12800, rotations=1), master_seed=1)
    dots, mls = O.synth_lanes(64, 12800, 1)
    hp, mp = _payloads(dots, mls, P.MPC_LIFT, np.random.default_rng(0))
    with pytest.raises(P.ConfigError):
        sess.comparison_only([h[:-1] for h in hp], mp, 64)
    bad = [h.copy() for h in hp]
    bad[1][2] ^= 1  # party 2's prev copy of lane 0 no longer equals party 1's own
    with pytest.raises(P.InconsistentShareError):
        sess.comparison_only(bad, mp, 64)
