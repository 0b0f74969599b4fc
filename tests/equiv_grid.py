"""Loader for tests/golden/equiv_grid.npz (oracle/gen_equiv.py): the reference's
equivalence-grid instances (equiv_common.hpp), boundary instances and
test_engine.cpp's planted / complement / ml = 0 cases."""
import os

import numpy as np

PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "equiv_grid.npz")
KINDS = {0: "grid", 1: "boundary", 2: "planted", 3: "complement", 4: "ml0"}


def load():
    d = np.load(PATH)
    m = d["meta"]
    out = []
    for i in range(len(m)):
        l, s, off, wo, qo = (int(m[k][i]) for k in ("l", "s", "off", "woff", "qoff"))
        wl = (l + 63) // 64
        out.append(dict(kind=KINDS[int(m["kind"][i])], backend=int(m["backend"][i]), variant=int(m["variant"][i]),
                        l=l, s=s, seed=int(m["seed"][i]), ratio=float(m["ratio"][i]), want=int(m["want"][i]),
                        got=int(m["got"][i]),
                        db_codes=d["db_codes"][wo:wo + s * wl].reshape(s, wl),
                        db_masks=d["db_masks"][wo:wo + s * wl].reshape(s, wl),
                        q_code=d["q_codes"][qo:qo + wl].reshape(1, wl),
                        q_mask=d["q_masks"][qo:qo + wl].reshape(1, wl),
                        ref_row_bits=d["ref_row_bits"][off:off + s]))
    return out


def plain_bits(inst):
    """tests/oracle.hpp:35-57 per row, in numpy (bit loop)."""
    l = inst["l"]
    a = min(1 << 16, int(np.floor((1 - 2 * inst["ratio"]) * (1 << 16) + 0.5)))
    b = 1 << 16
    out = []
    for r in range(inst["s"]):
        ml = hd = 0
        for w in range((l + 63) // 64):
            nb = min(64, l - 64 * w)
            mk = (1 << nb) - 1
            mm = int(inst["q_mask"][0, w]) & int(inst["db_masks"][r, w]) & mk
            ml += bin(mm).count("1")
            hd += bin((int(inst["q_code"][0, w]) ^ int(inst["db_codes"][r, w])) & mm).count("1")
        dot = ml - 2 * hd
        if inst["variant"] == 0:
            out.append(int(dot > int(np.ceil((1 - 2 * inst["ratio"]) * ml))))
        else:
            out.append(int(b * dot > a * ml))
    return np.array(out, np.uint8)
