"""bench.py's host-side accounting (no GPU): the per-lane work figures behind
`roofline` and `roofline_compare`, checked against SURVEY §8d / A.3 and the
reference's own PRF draw counts (the oracle's stream positions)."""
import importlib.util
import os

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench():
    spec = importlib.util.spec_from_file_location("bench", os.path.join(ROOT, "bench.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def test_int8_ops_per_lane_match_survey():
    b = _bench()
    # 460,800 int8 ops per comparison lane (mpc-lift, Shamir), 921,600 replicated
    assert b.ops_per_lane(1, 1) == 460_800
    assert b.ops_per_lane(0, 1) == 921_600
    # DESIGN §4 per-variant table (Shamir)
    assert b.ops_per_lane(1, 0) == 256_000
    assert b.ops_per_lane(1, 2) == 998_400
    assert b.ops_per_lane(1, 3) == 1_536_000


def test_prf_blocks_per_lane_match_reference_draws():
    """2.48 ChaCha12 blocks per lane (mpc-lift): the reference's draw count for n
    lanes is 2n + 125 W (+2n on seed 1, +6n on seed 3), SURVEY A.3."""
    b = _bench()
    n = 1 << 20
    W = n // 64
    draws = (2 * n + 125 * W) * 3 + 2 * n + 6 * n
    assert b.prf_blocks_per_lane(1) == pytest.approx(draws / 8 / n)
    assert b.prf_blocks_per_lane(1) == pytest.approx(2.482421875)
    # no-lift / const-lift: reshare of two dots + msb<32> (61 gates); plain-mask: hd + msb<16> (29)
    assert b.prf_blocks_per_lane(3) == pytest.approx((6 * n + 61 * W * 3) / 8 / n)
    assert b.prf_blocks_per_lane(0) == pytest.approx((3 * n + 29 * W * 3) / 8 / n)


def test_prf_blocks_match_oracle_stream_positions():
    """The same accounting from the oracle's PRF stream positions after one
    query (n a multiple of 64 lanes, so the figure is exact)."""
    from oracle import pyoracle as O
    b = _bench()
    l, s, persons = 128, 256, 1
    rng = O.Rng(3)
    dc, dm = O.records(rng, l, s, 0.9)
    qc, qm = O.records(rng, l, 2 * persons, 0.9)
    out = O.run_local(O.make_config(O.SHAMIR, l, 0.375, 31, False), 5, dc, dm, qc, qm, persons)
    n = int(O.lib().orc_lane_count(persons, s, 31, 0))
    assert n % 64 == 0
    W = n // 64
    pos = [int(x) for x in np.asarray(out.stream_pos).ravel()[:3]]
    assert pos[0] - pos[1] == 2 * n and pos[2] - pos[1] == 6 * n  # bit_inject draws (seed 1, seed 3)
    or_words = pos[1] - (2 * n + 125 * W)  # reshare + 125 AND gates, then the OR tree
    assert 0 < or_words < 2 * W  # halving tree: about W words over all levels
    assert (sum(pos) - 3 * or_words) / 8 / n == pytest.approx(b.prf_blocks_per_lane(1))


def test_compare_roofline_fields():
    """Per-kernel serial times of one profiled query -> ChaCha12 rates; the chain
    fraction = ChaCha floor / serial chain time."""
    b = _bench()
    lanes = 10_000_000
    prof = {"k_gate_keystream": (2.0, 4), "k_reshare": (3.0, 4), "k_lift": (1.0, 4), "k_inject": (2.5, 4),
            "k_msb": (1.5, 4), "k_limb_gemm_pair (hd)": (9.0, 8)}
    r = b.compare_roofline(prof, lanes, 1, {"hbm_gbs": 6500.0})
    assert set(r["kernels"]) == set(b.THRESHOLD_KERNELS)
    ks = r["kernels"]["k_reshare"]
    assert ks["chacha_blocks_per_s"] == pytest.approx(0.75 * lanes / 3e-3)
    assert r["kernels"]["k_inject"]["chacha_blocks_per_lane"] == 1.0
    assert r["kernels"]["k_gate_keystream"]["chacha_blocks_per_lane"] == pytest.approx(375 / 512)
    tot = sum(b.kernel_blocks_per_lane(k, 1) for k in b.THRESHOLD_KERNELS)
    assert tot == pytest.approx(b.prf_blocks_per_lane(1))  # the kernels account for every reference draw
    assert r["chain"]["serial_ms"] == pytest.approx(10.0)
    if r["chain"]["chacha_peak_blocks_per_s"]:
        floor = b.prf_blocks_per_lane(1) * lanes / r["chain"]["chacha_peak_blocks_per_s"] * 1e3
        assert r["chain"]["frac"] == pytest.approx(floor / 10.0)


def test_workload_labels_name_baseline_configs():
    b = _bench()
    assert b.workload_name(1_000_000, 32, 1) == "configs[2]"
    assert b.workload_name(100_000, 16, 1) == "configs[1]"
    assert b.workload_name(10_000, 1, 1) == "configs[0]"
    assert b.workload_name(1_000_000, 32, 4).startswith("configs[3]")
    assert b.workload_name(5_000, 3, 1) == "custom shape"
    assert b.ROWS_PER_GPU == 1_000_000 and b.PERSONS == 32 and b.REF_ROWS == 1_000


def test_both_arms_print_the_same_config():
    """--impl reference times a bounded row sample of the GPU arm's workload and
    prints the GPU arm's config, so the driver compares like with like."""
    import argparse
    b = _bench()
    args = argparse.Namespace(variant="mpc-lift", backend="shamir", rows=1_000_000, persons=32)
    c = b.arm_config(args, 1, 1_000_000, 32)
    assert c["workload"].startswith("configs[2]") and c["codes"] == 64 and c["db_rows_total"] == 1_000_000
    assert "153.6 KB/row" in c["l2"]
    src = open(b.__file__).read()
    assert src.count("\"config\": arm_config(args, world, args.rows") == 2  # the GPU arm and the reference arm
