"""The OR tree share for share: the GPU's or_tree_batch (csrc/ortree.cu) and the
C restatement (oracle/irismpc_oracle.c or_tree_groups) against the reference's
own or_tree_batch (include/irismpc/circuits.hpp:387-434, run by oracle/_ref
inside run_parties).  The aggregate components -- each party's own share of
every group's OR, before the open -- must be identical, not only the opened
bits."""
import numpy as np
import pytest

from oracle import pyoracle as O

needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built (no /root/reference here)")


def _gpu_ok():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


gpu = pytest.mark.gpu
needs_gpu = pytest.mark.skipif(not _gpu_ok(), reason="needs a B200")

SHAPES = [[1], [2], [3], [63], [64], [65], [127, 128, 129], [1000, 1, 7, 300], [0, 5, 0],
          [5000, 5000, 5000], [62 + 124 * 3] * 4, [4097] * 9]


@needs_ref
@pytest.mark.parametrize("lens", SHAPES, ids=lambda x: "-".join(map(str, x[:4])))
def test_restated_or_tree_equals_reference(lens):
    rng = np.random.default_rng(sum(lens) + len(lens))
    comps = rng.integers(0, 2, (3, sum(lens)), dtype=np.uint8)
    for seed in (77, 5001):
        agg, pos = O.or_tree_batch(O.party_seeds(seed), lens, comps)
        ref = O.ref_or_tree_batch_shares(lens, comps, seed)
        np.testing.assert_array_equal(agg, ref)
        # each level draws ceil(nb/64) words per group, every seed the same count
        assert pos[0] == pos[1] == pos[2]


def test_or_tree_opens_to_plain_or():
    rng = np.random.default_rng(9)
    lens = [10, 300, 1, 70]
    comps = rng.integers(0, 2, (3, sum(lens)), dtype=np.uint8)
    plain = comps[0] ^ comps[1] ^ comps[2]
    agg, _ = O.or_tree_batch(O.party_seeds(3), lens, comps)
    off = 0
    for g, n in enumerate(lens):
        assert (agg[0, g] ^ agg[1, g] ^ agg[2, g]) == int(plain[off:off + n].any())
        off += n


def _components(payloads, n):
    """party payloads of (own u64, prev u64) per 64-lane word -> component bits [3][n]"""
    out = np.zeros((3, n), np.uint8)
    for p in range(3):
        own = np.frombuffer(payloads[p].tobytes(), np.uint64).reshape(-1, 2)[:, 0].copy()
        out[p] = np.unpackbits(own.view(np.uint8), bitorder="little")[:n]
    return out


@gpu
@needs_gpu
@pytest.mark.parametrize("n", [1, 2, 65, 1000, 100_003, 3_000_001])
def test_gpu_or_tree_only_shares_equal_reference(n):
    """irismpc_gpu_or_tree_only (party_or_tree_only, engine.cpp:517-532): the
    aggregate components equal the reference's for the same sharing."""
    import paper_2405_04463_b200 as P
    rng = np.random.default_rng(n)
    bits = (rng.random(n) < 2.0 / n).astype(np.uint8)
    pay = P.share_bit_words(bits, rng)
    sess = P.Session(P.EngineConfig(backend=P.REPLICATED, l=12800, rotations=1), master_seed=5001)
    opened = sess.or_tree_only(pay, n)
    assert opened == int(bits.any())
    agg = sess.read_tap(P.TAP_AGG, 1)
    comps = _components(pay, n)
    want = (O.ref_or_tree_batch_shares([n], comps, 5001) if O.ref_available() and n <= 100_003
            else O.or_tree_batch(O.party_seeds(5001), [n], comps)[0])
    np.testing.assert_array_equal(agg, want)


@gpu
@needs_gpu
@pytest.mark.parametrize("be,var,l,s,persons,r,membership", [
    (O.SHAMIR, 1, 12800, 300, 3, 31, False),
    (O.REPLICATED, 1, 256, 2500, 5, 5, False),
    (O.SHAMIR, 3, 128, 1, 4, 31, False),       # one DB row, no-lift
    (O.REPLICATED, 0, 128, 0, 5, 31, False),   # empty DB: pair lanes only, plain-mask
    (O.SHAMIR, 1, 256, 777, 1, 7, False),      # one person: no pair lanes
    (O.SHAMIR, 2, 256, 4099, 1, 1, True),      # membership: one group of every row
    (O.REPLICATED, 1, 128, 1, 1, 1, True),     # one lane
    (O.SHAMIR, 1, 128, 50, 40, 3, False),      # 40 persons: pair lanes dominate, many pair blocks per group
    (O.REPLICATED, 2, 64, 100, 9, 31, False),  # pair blocks of 124 lanes straddling 64-lane words
])
def test_gpu_batch_query_or_tree_shares_equal_oracle(be, var, l, s, persons, r, membership):
    """The batch query's aggregate components (groups = Schedule::groups,
    engine.cpp:221-289: a person's DB lanes, then its pair lanes) equal the
    oracle's, whose tree is pinned to the reference above."""
    import paper_2405_04463_b200 as P
    seed = 300 + s + persons
    rng = O.Rng(seed)
    dc, dm = O.records(rng, l, s, 0.9)
    qc, qm = O.records(rng, l, 1 if membership else 2 * persons, 0.9)
    if s:
        qc[0], qm[0] = dc[s // 2], dm[s // 2]
    cfg = P.EngineConfig(backend=be, l=l, rotations=r, variant=var)
    m, sess = P.run_batch_local(cfg, qc, qm, dc, dm, seed, persons=persons, membership=membership)
    ref = O.run_local(O.make_config(be, l, 0.375, r, variant=var), seed, dc, dm, qc, qm, persons,
                      membership=membership)
    groups = 1 if membership else persons
    np.testing.assert_array_equal(sess.read_tap(P.TAP_AGG, groups), ref.agg)
    np.testing.assert_array_equal(m, ref.person_match)
    np.testing.assert_array_equal(sess.stream_positions(), ref.stream_pos)
