"""Generates tests/golden/equiv_grid.npz from the REFERENCE (oracle/_ref):
the randomized equivalence grid of /root/reference/proj/tests/equiv_common.hpp
(run_instance, :61-89) over both backends x 4 variants x l in {8, 64, 128} x
s in {1, 4, 64} (25 seeds at ratio 0.375, 3 at 0.3; the reference's C1 runs
100 seeds at l in {8, 64}), its 100 threshold-boundary instances
(run_boundary_instances, :93-128), and test_engine.cpp's planted / complement /
ml = 0 cases (:42-82).  For every instance it stores the records, the
plaintext oracle's answer (oracle::naive_membership), the reference's own
3-party result and its debug row bits.  Test infrastructure only; run it where
/root/reference was built into oracle/_ref:

    python oracle/gen_equiv.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle import pyoracle as O  # noqa: E402

OUT = os.path.join(os.path.dirname(HERE), "tests", "golden", "equiv_grid.npz")


def main():
    meta, dbc, dbm, qcs, qms, rbits = [], [], [], [], [], []
    off = woff = qoff = 0

    def add(kind, be, va, l, s, seed, ratio, dc, dm, qc, qm, want, got, rb):
        nonlocal off, woff, qoff
        wl = O.words(l)
        meta.append((kind, be, va, l, s, seed, ratio, want, got, off, woff, qoff))
        dbc.append(np.asarray(dc, np.uint64).reshape(s, wl).ravel())
        dbm.append(np.asarray(dm, np.uint64).reshape(s, wl).ravel())
        qcs.append(np.asarray(qc, np.uint64).ravel()[:wl])
        qms.append(np.asarray(qm, np.uint64).ravel()[:wl])
        rbits.append(np.asarray(rb, np.uint8).ravel()[:s] if rb is not None else np.full(s, 255, np.uint8))
        off += s
        woff += s * wl
        qoff += wl

    for ratio, nseeds in ((0.375, 25), (0.3, 3)):
        for be in (0, 1):
            for va in (0, 1, 2, 3):
                for l in (8, 64, 128):
                    for s in (1, 4, 64):
                        for seed in range(1, nseeds + 1):
                            dc, dm, qc, qm, want, got, rb = O.ref_equiv_instance(be, va, l, s, seed, ratio)
                            add(0, be, va, l, s, seed, ratio, dc, dm, qc, qm, want, got, rb)
    b = O.ref_boundary_instances(100)
    for i in range(100):
        add(1, int(b["backend"][i]), int(b["variant"][i]), 64, 1, int(b["seed"][i]), float(b["ratio"][i]),
            b["row_code"][i:i + 1], b["row_mask"][i:i + 1], b["q_code"][i:i + 1], b["q_mask"][i:i + 1],
            int(b["want"][i]), int(b["got"][i]), None)
    for which in (0, 1, 2):
        for be in (0, 1):
            for va in (0, 1, 2, 3):
                dc, dm, qc, qm, want, got = O.ref_engine_case(which, be, va)
                add(2 + which, be, va, 64, dc.shape[0], 500 + which, 0.375, dc, dm, qc, qm, want, got, None)
    m = np.array(meta, dtype=[("kind", "i4"), ("backend", "i4"), ("variant", "i4"), ("l", "i4"), ("s", "i4"),
                              ("seed", "u8"), ("ratio", "f8"), ("want", "u1"), ("got", "u1"), ("off", "u8"),
                              ("woff", "u8"), ("qoff", "u8")])
    np.savez_compressed(OUT, meta=m, db_codes=np.concatenate(dbc), db_masks=np.concatenate(dbm),
                        q_codes=np.concatenate(qcs), q_masks=np.concatenate(qms), ref_row_bits=np.concatenate(rbits))
    print(f"{len(meta)} instances, {int((m['want'] != m['got']).sum())} reference mismatches -> {OUT}")


if __name__ == "__main__":
    main()
