"""The reference's equivalence grid as committed fixtures (CPU): the reference
passes its own grid (got == want), the numpy plaintext predicate agrees with
the reference's oracle, and the C restatement (oracle/) reproduces every
opened aggregate and row bit.  tests/test_gpu_equivalence.py runs the same
instances through the B200."""
import numpy as np
import pytest

from oracle import pyoracle as O
from equiv_grid import load, plain_bits

INST = load()


def test_grid_shape_and_reference_passes_its_own_grid():
    kinds = {}
    for x in INST:
        kinds[x["kind"]] = kinds.get(x["kind"], 0) + 1
    assert kinds == {"grid": 2016, "boundary": 100, "planted": 8, "complement": 8, "ml0": 8}
    assert all(x["got"] == x["want"] for x in INST)
    assert {x["l"] for x in INST if x["kind"] == "grid"} == {8, 64, 128}
    # the grid exercises both outcomes, empty / full masks and the boundary
    assert 0.3 < np.mean([x["want"] for x in INST if x["kind"] == "grid"]) < 0.7
    assert any((x["db_masks"] == 0).all(1).any() for x in INST if x["kind"] == "grid")
    assert all(x["want"] == 1 for x in INST if x["kind"] == "planted")
    assert all(x["want"] == 0 for x in INST if x["kind"] in ("complement", "ml0"))


@pytest.mark.parametrize("chunk", range(4))
def test_oracle_restatement_on_grid(chunk):
    for x in INST[chunk::4]:
        bits = plain_bits(x)
        assert int(bits.any()) == x["want"]
        if x["kind"] == "grid":
            np.testing.assert_array_equal(bits, x["ref_row_bits"])
        cfg = O.make_config(x["backend"], x["l"], x["ratio"], 1, True, variant=x["variant"])
        r = O.run_local(cfg, x["seed"], x["db_codes"], x["db_masks"], x["q_code"], x["q_mask"], 1, membership=True)
        assert int(r.person_match[0]) == x["want"], x
        np.testing.assert_array_equal(r.row_bits, bits)
