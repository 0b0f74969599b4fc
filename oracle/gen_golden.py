"""Generate tests/golden/ref_vectors.json from the REFERENCE itself.

TEST INFRASTRUCTURE.  Runs only where oracle/_ref/libirismpc_ref.so was built
from /root/reference (`make -C oracle ref`).  Every expected value below comes
from a reference entry point (ref_driver.cpp -> unmodified reference code); the
C restatement is NOT used to produce expectations, only to regenerate inputs
whose generator (Rng / random_record) is itself pinned by the KATs recorded
here.

    python oracle/gen_golden.py
"""
from __future__ import annotations

import ctypes as C
import hashlib
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import pyoracle as O  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                   "ref_vectors.json")

# (backend, l, s, persons, rotations, seed, membership, ratio, planted[, variant])
# variant defaults to mpc-lift (the north-star path); the tail covers the
# other three variants (shares.hpp:28) on both backends.
CASES = [
    (0, 64, 4, 1, 1, 101, True, 0.375, True),
    (1, 64, 4, 1, 1, 102, True, 0.375, True),
    (0, 8, 3, 1, 1, 103, True, 0.375, False),
    (1, 8, 5, 1, 1, 104, True, 0.375, False),
    (0, 64, 64, 1, 1, 105, True, 0.3, True),
    (1, 64, 64, 1, 1, 106, True, 0.3, False),
    (0, 128, 3, 3, 3, 107, False, 0.375, True),
    (1, 128, 3, 3, 3, 108, False, 0.375, True),
    (0, 128, 0, 4, 31, 109, False, 0.2, False),
    (1, 256, 7, 2, 31, 110, False, 0.375, True),
    (0, 256, 9, 2, 31, 111, False, 0.375, False),
    (1, 12800, 2, 1, 31, 112, False, 0.375, True),
    (0, 12800, 3, 1, 31, 113, False, 0.375, True),
    (1, 12800, 40, 2, 31, 114, False, 0.375, True),
] + [
    (be, l, s, persons, r, 200 + 10 * var + 2 * i + be, memb, ratio, planted, var)
    for var in (O.PLAIN_MASK, O.CONST_LIFT, O.NO_LIFT)
    for i, (l, s, persons, r, memb, ratio, planted) in enumerate([
        (64, 6, 1, 1, True, 0.375, True),
        (128, 3, 3, 3, False, 0.375, True),
        (256, 9, 2, 31, False, 0.3, False),
        (12800, 3, 1, 31, False, 0.375, True),
    ])
    for be in (0, 1)
]


def sha(a: np.ndarray) -> str:
    """sha256 of the little-endian bytes at the array's ring width (u16 / u32 / i64)."""
    dt = {np.dtype(np.uint16): "<u2", np.dtype(np.uint32): "<u4", np.dtype(np.int64): "<i8"}[a.dtype]
    return hashlib.sha256(np.ascontiguousarray(a).astype(dt).tobytes()).hexdigest()


def inputs(l, s, persons, seed, membership, planted):
    """Synthetic records: Rng(seed) draws s DB rows then the query codes."""
    rng = O.Rng(seed)
    dc, dm = O.records(rng, l, s, 0.85)
    nq = 1 if membership else 2 * persons
    qc, qm = O.records(rng, l, nq, 0.85)
    if planted and s > 0:
        qc[0] = dc[s // 2]
        qm[0] = dm[s // 2]
    return dc, dm, qc, qm


FILES = os.path.join(os.path.dirname(OUT), "files")


def gen_files():
    """Reference-written IRMP / IRSD / IRS1 files (io.cpp) for the file-format tests:
    the `irismpc share` dealer over a 3-row l=64 DB, seed 9, every variant (Shamir)
    plus replicated mpc-lift."""
    os.makedirs(FILES, exist_ok=True)
    l, s, seed = 64, 3, 9
    dc, dm = O.records(O.Rng(31), l, s, 0.85)
    db = os.path.join(FILES, "db.irmp")
    O.ref_write_iris_db(db, dc, dm, l)
    out = {"db": "db.irmp", "l": l, "s": s, "records_rng": 31, "seed": seed, "shares": []}
    for be, var in [(1, 0), (1, 1), (1, 2), (1, 3), (0, 1)]:
        names = [f"db.b{be}.v{var}.p{p}.irs" for p in (1, 2, 3)]
        seeds = [f"seeds.b{be}.v{var}.p{p}.irsd" for p in (1, 2, 3)]
        O.ref_share_files(db, be, var, seed, [os.path.join(FILES, n) for n in names],
                          [os.path.join(FILES, n) for n in seeds])
        out["shares"].append({"backend": be, "variant": var, "files": names, "seed_files": seeds})
    return out


def main():
    R = O.ref()
    g = {"generated_by": "oracle/gen_golden.py from oracle/_ref (reference compiled from /root/reference/proj)"}

    s42 = np.zeros(16, np.uint8)
    R.ref_seed_from_u64(42, O._p(s42, O.u8p))
    blk = np.zeros(16, np.uint32)
    R.ref_chacha_block(O._p(s42, O.u8p), 0, 0, O._p(blk, O.u32p))
    blk5 = np.zeros(16, np.uint32)
    R.ref_chacha_block(O._p(s42, O.u8p), 5, 3, O._p(blk5, O.u32p))
    ps = np.zeros(48, np.uint8)
    R.ref_party_seeds(7, O._p(ps, O.u8p))
    lam = np.zeros(6, np.uint16)
    R.ref_lambda16(O._p(lam, O.u16p))
    rng_draws = np.zeros(20, np.uint64)
    R.ref_rng_u64(2, 20, O._p(rng_draws, O.u64p))
    g["prf"] = {
        "seed_from_u64_42": bytes(s42).hex(),
        "chacha12_seed42_block0_stream0": [int(x) for x in blk],
        "chacha12_seed42_block5_stream3": [int(x) for x in blk5],
        "party_seeds_7": bytes(ps).hex(),
        "rng2_first20": [str(int(x)) for x in rng_draws],
    }
    g["lambda16"] = [int(x) for x in lam]

    # random_record(l, Rng(11), density) sequence
    dens = np.array([0.85, 0.9, 0.0, 1.0, 0.3], np.float64)
    l = 128
    rc = np.zeros((5, 2), np.uint64)
    rm = np.zeros((5, 2), np.uint64)
    R.ref_random_records(11, l, 5, dens.ctypes.data_as(C.POINTER(C.c_double)), O._p(rc, O.u64p), O._p(rm, O.u64p))
    g["random_records_rng11_l128"] = {"density": dens.tolist(), "code": [[str(int(w)) for w in r] for r in rc],
                                      "mask": [[str(int(w)) for w in r] for r in rm]}

    # dealer payload hashes
    deals = []
    for be in (0, 1):
        for l in (64, 12800):
            dc, dm = rc[:3, :1] if l == 64 else None, None
            rng = O.Rng(21)
            dc, dm = O.records(rng, l, 3, 0.9)
            rb = O.record_bytes(be, l)
            outs = [np.zeros(3 * rb, np.uint8) for _ in range(3)]
            R.ref_deal(be, O.MPC_LIFT, l, 7, 1, 3, O._p(dc, O.u64p), O._p(dm, O.u64p), *[O._p(x, O.u8p) for x in outs])
            deals.append({"backend": be, "l": l, "records_rng": 21, "nrec": 3, "deal_seed": 7, "tag": 1,
                          "sha256": [hashlib.sha256(x.tobytes()).hexdigest() for x in outs],
                          "head_hex": [x[:32].tobytes().hex() for x in outs]})
    for var in (O.PLAIN_MASK, O.CONST_LIFT, O.NO_LIFT):
        for be in (0, 1):
            l = 128
            rng = O.Rng(21)
            dc, dm = O.records(rng, l, 3, 0.9)
            rb = O.record_bytes(be, l, var)
            outs = [np.zeros(3 * rb, np.uint8) for _ in range(3)]
            R.ref_deal(be, var, l, 7, 1, 3, O._p(dc, O.u64p), O._p(dm, O.u64p), *[O._p(x, O.u8p) for x in outs])
            deals.append({"backend": be, "variant": var, "l": l, "records_rng": 21, "nrec": 3, "deal_seed": 7,
                          "tag": 1, "sha256": [hashlib.sha256(x.tobytes()).hexdigest() for x in outs],
                          "head_hex": [x[:32].tobytes().hex() for x in outs]})
    g["deal"] = deals
    lam32 = O.lambda_k(32)
    g["lambda32_restated"] = [int(x) for x in lam32]

    cases = []
    for spec in CASES:
        (be, l, s, persons, r, seed, membership, ratio, planted), var = spec[:9], (spec[9] if len(spec) > 9 else O.MPC_LIFT)
        dc, dm, qc, qm = inputs(l, s, persons, seed, membership, planted)
        res = O.ref_run_local(be, l, ratio, r, seed, dc, dm, qc, qm, persons, membership, debug_rows=True,
                              variant=var)
        db = O.deal(be, l, dc, dm, O.Rng(sub=(seed, 1)), variant=var)
        q = O.deal(be, l, qc, qm, O.Rng(sub=(seed, 2)), variant=var)
        # the dealt payloads must equal the reference dealer's (pinned above) — recheck here
        outs = [np.zeros(max(1, s * O.record_bytes(be, l, var)), np.uint8) for _ in range(3)]
        if s:
            R.ref_deal(be, var, l, seed, 1, s, O._p(dc, O.u64p), O._p(dm, O.u64p), *[O._p(x, O.u8p) for x in outs])
            assert all((a == b[: len(a)]).all() for a, b in zip(db, outs))
        seeds = O.party_seeds(seed)
        dh, dmm, rh, rm = O.ref_dots_reshare(be, l, r, seeds, db, s, q, persons, membership, variant=var)
        n = int(res["lanes"])
        case = {
            "backend": be, "l": l, "s": s, "persons": persons, "rotations": r, "seed": seed,
            "membership": membership, "ratio": ratio, "planted": planted, "lanes": n,
            "person_match": [int(x) for x in res["person_match"]],
            "row_bits_hex": np.packbits(res["row_bits"], bitorder="little").tobytes().hex(),
            "stats": res["stats"],
            "sha256": {"dot_hd": sha(dh), "rs_hd": sha(rh)},
        }
        if var != O.MPC_LIFT:
            case["variant"] = var
        if O.mask_bits(var):
            case["sha256"].update(dot_ml=sha(dmm), rs_ml=sha(rm))
        else:
            case["sha256"]["public_ml"] = sha(O.ref_dots_reshare.public_ml)
        if n <= 64:
            case["dot_hd"] = dh.tolist()
            case["rs_hd"] = rh.tolist()
            if O.mask_bits(var):
                case["dot_ml"] = dmm.tolist()
                case["rs_ml"] = rm.tolist()
            else:
                case["public_ml"] = O.ref_dots_reshare.public_ml.tolist()
        cases.append(case)
        print(f"case var={var} be={be} l={l} s={s} persons={persons} r={r} lanes={n} match={case['person_match']}")
    g["cases"] = cases
    g["files"] = gen_files()
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    with open(OUT, "w") as f:
        json.dump(g, f, indent=1)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
