"""ctypes bindings for the test-side checkers (TEST INFRASTRUCTURE ONLY).

Loaded only by tests/, ``__graft_entry__.smoke()`` and bench.py's
``cpu_baseline`` / ``--impl reference`` legs.  Two libraries:

* ``liboracle.so`` — the C restatement (oracle/irismpc_oracle.c), always built;
* ``_ref/libirismpc_ref.so`` — the reference compiled from /root/reference by
  oracle/Makefile (present only where that tree existed at build time).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libirismpc_ref.so")

REPLICATED, SHAMIR = 0, 1
PLAIN_MASK, MPC_LIFT, CONST_LIFT, NO_LIFT = 0, 1, 2, 3
VARIANT_NAMES = {"plain-mask": PLAIN_MASK, "mpc-lift": MPC_LIFT, "const-lift": CONST_LIFT, "no-lift": NO_LIFT}

u8p = C.POINTER(C.c_uint8)
u16p = C.POINTER(C.c_uint16)
u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)


def _p(a, t):
    return None if a is None else a.ctypes.data_as(t)


class OrcConfig(C.Structure):
    _fields_ = [("backend", C.c_int32), ("variant", C.c_int32), ("l", C.c_uint32), ("a", C.c_uint32),
                ("b", C.c_uint32), ("rotations", C.c_uint32), ("debug_rows", C.c_int32),
                ("ratio", C.c_double)]


class OrcStats(C.Structure):
    _fields_ = [(k, C.c_uint64) for k in (
        "dot_bytes", "lift_bytes", "msb_bytes", "or_tree_bytes",
        "dot_rounds", "lift_rounds", "msb_rounds", "or_tree_rounds")]


class OrcOut(C.Structure):
    _fields_ = [("person_match", u8p), ("row_bits", u8p), ("dot_hd", u32p), ("dot_ml", u32p),
                ("public_ml", C.POINTER(C.c_int64)), ("rs_hd", u32p), ("rs_ml", u32p), ("ml32", u32p),
                ("diff", u32p), ("msb", u8p), ("stream_pos", u64p), ("stats", C.POINTER(OrcStats)),
                ("agg", u8p)]


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} missing: run `make -C oracle`")
        L = C.CDLL(LIB_PATH)
        L.orc_chacha_block.argtypes = [u8p, C.c_uint64, C.c_uint64, u32p]
        L.orc_seed_from_u64.argtypes = [C.c_uint64, u8p]
        L.orc_derive.argtypes = [u8p, C.c_uint64, u8p]
        L.orc_stream_at.argtypes = [u8p, C.c_uint64, C.c_uint64]
        L.orc_stream_at.restype = C.c_uint64
        L.orc_party_seeds.argtypes = [C.c_uint64, u8p]
        L.orc_rng_new.argtypes = [C.c_uint64]
        L.orc_rng_new.restype = C.c_void_p
        L.orc_rng_sub.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_rng_sub.restype = C.c_void_p
        L.orc_rng_free.argtypes = [C.c_void_p]
        L.orc_rng_next.argtypes = [C.c_void_p]
        L.orc_rng_next.restype = C.c_uint64
        L.orc_rng_below.argtypes = [C.c_void_p, C.c_uint64]
        L.orc_rng_below.restype = C.c_uint64
        L.orc_rng_record.argtypes = [C.c_void_p, C.c_uint32, C.c_double, u64p, u64p]
        L.orc_lambda16.argtypes = [u16p]
        L.orc_lambda.argtypes = [C.c_uint, u32p]
        L.orc_code_record_bytes.argtypes = [C.c_int, C.c_int, C.c_uint32]
        L.orc_code_record_bytes.restype = C.c_size_t
        L.orc_mask_record_bytes.argtypes = [C.c_int, C.c_int, C.c_uint32]
        L.orc_mask_record_bytes.restype = C.c_size_t
        for f in ("orc_code_bits", "orc_mask_bits", "orc_cmp_bits"):
            getattr(L, f).argtypes = [C.c_int]
            getattr(L, f).restype = C.c_uint
        L.orc_deal_payload_v.argtypes = [C.c_int, C.c_int, C.c_uint32, C.c_uint64, u64p, u64p, C.c_void_p,
                                         u8p, u8p, u8p]
        L.orc_deal_payload.argtypes = [C.c_int, C.c_uint32, C.c_uint64, u64p, u64p, C.c_void_p,
                                       u8p, u8p, u8p]
        L.orc_lane_count.argtypes = [C.c_uint32, C.c_uint64, C.c_uint32, C.c_int]
        L.orc_lane_count.restype = C.c_uint64
        L.orc_query.argtypes = [C.POINTER(OrcConfig), u8p, u8p, u8p, u8p, C.c_uint64, u8p, u8p, u8p,
                                C.c_uint32, C.c_int, u64p, C.POINTER(OrcOut)]
        L.orc_run_local.argtypes = [C.POINTER(OrcConfig), C.c_uint64, C.c_uint64, u64p, u64p,
                                    C.c_uint32, u64p, u64p, C.c_int, C.POINTER(OrcOut)]
        L.orc_match_a.argtypes = [C.c_double]
        L.orc_match_a.restype = C.c_uint32
        L.orc_validate.argtypes = [C.POINTER(OrcConfig)]
        _lib = L
    return _lib


def ref_available() -> bool:
    return os.path.exists(REF_PATH)


def ref():
    global _ref
    if _ref is None:
        if not ref_available():
            raise RuntimeError(f"{REF_PATH} missing: run `make -C oracle ref` where /root/reference exists")
        R = C.CDLL(REF_PATH)
        R.ref_chacha_block.argtypes = [u8p, C.c_uint64, C.c_uint64, u32p]
        R.ref_seed_from_u64.argtypes = [C.c_uint64, u8p]
        R.ref_party_seeds.argtypes = [C.c_uint64, u8p]
        R.ref_rng_u64.argtypes = [C.c_uint64, C.c_uint64, u64p]
        R.ref_random_records.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.POINTER(C.c_double),
                                         u64p, u64p]
        R.ref_lambda16.argtypes = [u16p]
        R.ref_deal.argtypes = [C.c_int, C.c_int, C.c_uint32, C.c_uint64, C.c_uint64, C.c_uint64, u64p, u64p,
                               u8p, u8p, u8p]
        R.ref_deal.restype = C.c_uint64
        R.ref_run_local.argtypes = [C.c_int, C.c_int, C.c_uint32, C.c_double, C.c_uint32, C.c_int, C.c_int,
                                    C.c_uint64, C.c_uint64, u64p, u64p, C.c_uint32, u64p, u64p,
                                    C.c_int, u8p, u8p, u64p, C.POINTER(C.c_double), u64p]
        R.ref_dots_reshare.argtypes = [C.c_int, C.c_int, C.c_uint32, C.c_uint32, u8p, C.POINTER(u8p),
                                       C.c_uint64, C.POINTER(u8p), C.c_uint32, C.c_int,
                                       u32p, u32p, C.POINTER(C.c_int64), u32p, u32p]
        R.ref_write_iris_db.argtypes = [C.c_char_p, C.c_uint32, C.c_uint64, u64p, u64p]
        R.ref_share_files.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_uint64, C.c_char_p * 3, C.c_char_p * 3]
        R.ref_read_share_file.argtypes = [C.c_char_p, u32p, u64p, u64p]
        R.ref_bench_prepare.argtypes = [C.c_int, C.c_int, C.c_uint32, C.c_uint64, C.c_uint32]
        R.ref_bench_prepare.restype = C.c_void_p
        R.ref_bench_step.argtypes = [C.c_void_p, u8p]
        R.ref_bench_step.restype = C.c_double
        R.ref_bench_free.argtypes = [C.c_void_p]
        _ref = R
    return _ref


# ---------------------------------------------------------------- helpers

def words(l: int) -> int:
    return (l + 63) // 64


def record_bytes(backend: int, l: int, variant: int = MPC_LIFT) -> int:
    L = lib()
    return int(L.orc_code_record_bytes(backend, variant, l) + L.orc_mask_record_bytes(backend, variant, l))


def code_bits(variant: int) -> int:
    return int(lib().orc_code_bits(variant))


def mask_bits(variant: int) -> int:
    return int(lib().orc_mask_bits(variant))


def cmp_bits(variant: int) -> int:
    return int(lib().orc_cmp_bits(variant))


def party_seeds(master: int) -> np.ndarray:
    out = np.zeros(48, np.uint8)
    lib().orc_party_seeds(master, _p(out, u8p))
    return out


def chacha_block(seed: np.ndarray, block: int, stream: int = 0) -> np.ndarray:
    out = np.zeros(16, np.uint32)
    lib().orc_chacha_block(_p(np.ascontiguousarray(seed, np.uint8), u8p), block, stream, _p(out, u32p))
    return out


def seed_from_u64(v: int) -> np.ndarray:
    out = np.zeros(16, np.uint8)
    lib().orc_seed_from_u64(v, _p(out, u8p))
    return out


def lambda16() -> np.ndarray:
    out = np.zeros(6, np.uint16)
    lib().orc_lambda16(_p(out, u16p))
    return out


def lambda_k(K: int) -> np.ndarray:
    out = np.zeros(6, np.uint32)
    lib().orc_lambda(K, _p(out, u32p))
    return out


class Rng:
    """Rng(seed) of prf.hpp:138 (stream of u64 draws) — C restatement."""

    def __init__(self, seed: int | None = None, sub: tuple[int, int] | None = None):
        L = lib()
        self.h = L.orc_rng_sub(*sub) if sub is not None else L.orc_rng_new(seed)

    def __del__(self):
        try:
            lib().orc_rng_free(self.h)
        except Exception:
            pass

    def next(self) -> int:
        return int(lib().orc_rng_next(self.h))

    def below(self, bound: int) -> int:
        return int(lib().orc_rng_below(self.h, bound))

    def record(self, l: int, density: float):
        c = np.zeros(words(l), np.uint64)
        m = np.zeros(words(l), np.uint64)
        lib().orc_rng_record(self.h, l, density, _p(c, u64p), _p(m, u64p))
        return c, m


def records(rng: Rng, l: int, n: int, density: float = 0.9):
    codes = np.zeros((n, words(l)), np.uint64)
    masks = np.zeros((n, words(l)), np.uint64)
    for i in range(n):
        codes[i], masks[i] = rng.record(l, density)
    return codes, masks


def deal(backend: int, l: int, codes: np.ndarray, masks: np.ndarray, rng: Rng, variant: int = MPC_LIFT):
    """deal_db_payload / deal_query_payload -> three uint8 payloads."""
    n = codes.shape[0]
    rb = record_bytes(backend, l, variant)
    outs = [np.zeros(max(1, n * rb), np.uint8) for _ in range(3)]
    lib().orc_deal_payload_v(backend, variant, l, n, _p(np.ascontiguousarray(codes), u64p),
                             _p(np.ascontiguousarray(masks), u64p), rng.h,
                             *[_p(o, u8p) for o in outs])
    return [o[: n * rb] for o in outs]


@dataclass
class QueryResult:
    person_match: np.ndarray
    row_bits: np.ndarray | None = None
    dot_hd: np.ndarray | None = None
    dot_ml: np.ndarray | None = None
    public_ml: np.ndarray | None = None
    rs_hd: np.ndarray | None = None
    rs_ml: np.ndarray | None = None
    ml32: np.ndarray | None = None
    diff: np.ndarray | None = None
    msb: np.ndarray | None = None
    stream_pos: np.ndarray | None = None
    stats: list | None = None
    agg: np.ndarray | None = None  # [3][groups] OR-tree output components


def make_config(backend: int, l: int, ratio: float = 0.375, rotations: int = 31,
                debug_rows: bool = False, variant: int = MPC_LIFT) -> OrcConfig:
    L = lib()
    return OrcConfig(backend, variant, l, L.orc_match_a(ratio), 1 << 16, rotations, 1 if debug_rows else 0,
                     ratio)


def _alloc_out(n: int, ngroups: int, want_all: bool):
    arrs = dict(person_match=np.zeros(max(1, ngroups), np.uint8), row_bits=np.zeros(max(1, n), np.uint8),
                agg=np.zeros(3 * max(1, ngroups), np.uint8))
    if want_all:
        arrs.update({k: np.zeros(3 * max(1, n), np.uint32)
                     for k in ("dot_hd", "dot_ml", "rs_hd", "rs_ml", "ml32", "diff")})
        arrs.update(public_ml=np.zeros(max(1, n), np.int64), msb=np.zeros(3 * max(1, n), np.uint8))
    stats = (OrcStats * 3)()
    pos = np.zeros(3, np.uint64)
    out = OrcOut(_p(arrs["person_match"], u8p), _p(arrs["row_bits"], u8p),
                 _p(arrs.get("dot_hd"), u32p), _p(arrs.get("dot_ml"), u32p),
                 _p(arrs.get("public_ml"), C.POINTER(C.c_int64)),
                 _p(arrs.get("rs_hd"), u32p), _p(arrs.get("rs_ml"), u32p),
                 _p(arrs.get("ml32"), u32p), _p(arrs.get("diff"), u32p), _p(arrs.get("msb"), u8p),
                 _p(pos, u64p), C.cast(stats, C.POINTER(OrcStats)), _p(arrs["agg"], u8p))
    return out, arrs, stats, pos


def _width_dtype(bits: int):
    return np.uint16 if bits == 16 else np.uint32


def _finish(arrs, stats, pos, n, ngroups, want_all, debug_rows, variant=MPC_LIFT):
    res = QueryResult(person_match=arrs["person_match"][:ngroups].copy(),
                      agg=arrs["agg"][: 3 * ngroups].reshape(3, ngroups).copy())
    if debug_rows:
        res.row_bits = arrs["row_bits"][:n].copy()
    if want_all:
        # dot / reshare arrays in their ring's width (u16 for 16-bit rings)
        kh, km = code_bits(variant), mask_bits(variant)
        widths = dict(dot_hd=kh, rs_hd=kh, dot_ml=km or 16, rs_ml=km or 16, ml32=32,
                      diff=cmp_bits(variant))
        for k, bits in widths.items():
            setattr(res, k, arrs[k][: 3 * n].reshape(3, n).astype(_width_dtype(bits)))
        res.msb = arrs["msb"][: 3 * n].reshape(3, n).copy()
        if km == 0:
            res.public_ml = arrs["public_ml"][:n].copy()
    res.stream_pos = pos.copy()
    res.stats = [{f: getattr(stats[p], f) for f, _ in OrcStats._fields_} for p in range(3)]
    return res


def query(cfg: OrcConfig, seeds: np.ndarray, db: list, s: int, q: list, persons: int,
          membership: bool = False, want_all: bool = False, stream_start=None) -> QueryResult:
    L = lib()
    n = int(L.orc_lane_count(persons, s, cfg.rotations, 1 if membership else 0))
    ngroups = 1 if membership else persons
    out, arrs, stats, pos = _alloc_out(n, ngroups, want_all)
    ss = None if stream_start is None else np.ascontiguousarray(stream_start, np.uint64)
    dbb = [np.ascontiguousarray(x, np.uint8) if len(x) else np.zeros(1, np.uint8) for x in db]
    qb = [np.ascontiguousarray(x, np.uint8) for x in q]
    rc = L.orc_query(C.byref(cfg), _p(np.ascontiguousarray(seeds, np.uint8), u8p),
                     *[_p(x, u8p) for x in dbb], s, *[_p(x, u8p) for x in qb], persons,
                     1 if membership else 0, _p(ss, u64p), C.byref(out))
    if rc:
        raise RuntimeError(f"orc_query failed with status {rc}")
    return _finish(arrs, stats, pos, n, ngroups, want_all, cfg.debug_rows, cfg.variant)


def run_local(cfg: OrcConfig, seed: int, db_codes, db_masks, q_codes, q_masks, persons: int,
              membership: bool = False, want_all: bool = False) -> QueryResult:
    L = lib()
    s = db_codes.shape[0]
    n = int(L.orc_lane_count(persons, s, cfg.rotations, 1 if membership else 0))
    ngroups = 1 if membership else persons
    out, arrs, stats, pos = _alloc_out(n, ngroups, want_all)
    dc = np.ascontiguousarray(db_codes if s else np.zeros((1, words(cfg.l)), np.uint64))
    dm = np.ascontiguousarray(db_masks if s else np.zeros((1, words(cfg.l)), np.uint64))
    rc = L.orc_run_local(C.byref(cfg), seed, s, _p(dc, u64p), _p(dm, u64p), persons,
                         _p(np.ascontiguousarray(q_codes), u64p), _p(np.ascontiguousarray(q_masks), u64p),
                         1 if membership else 0, C.byref(out))
    if rc:
        raise RuntimeError(f"orc_run_local failed with status {rc}")
    return _finish(arrs, stats, pos, n, ngroups, want_all, cfg.debug_rows, cfg.variant)


# ------------------------------------------------------- the reference (_ref)

def ref_run_local(backend: int, l: int, ratio: float, rotations: int, seed: int, db_codes, db_masks,
                  q_codes, q_masks, persons: int, membership: bool = False, debug_rows: bool = False,
                  parallel_dot: bool = True, variant: int = MPC_LIFT):
    R = ref()
    s = db_codes.shape[0]
    n = int(lib().orc_lane_count(persons, s, rotations, 1 if membership else 0))
    ngroups = 1 if membership else persons
    pm = np.zeros(max(1, ngroups), np.uint8)
    rb = np.zeros(max(1, n), np.uint8)
    st = np.zeros(24, np.uint64)
    wall = C.c_double(0)
    lanes = C.c_uint64(0)
    dc = np.ascontiguousarray(db_codes if s else np.zeros((1, words(l)), np.uint64))
    dm = np.ascontiguousarray(db_masks if s else np.zeros((1, words(l)), np.uint64))
    rc = R.ref_run_local(backend, variant, l, ratio, rotations, 1 if debug_rows else 0, 1 if parallel_dot else 0,
                         seed, s, _p(dc, u64p), _p(dm, u64p), persons,
                         _p(np.ascontiguousarray(q_codes), u64p), _p(np.ascontiguousarray(q_masks), u64p),
                         1 if membership else 0, _p(pm, u8p), _p(rb, u8p), _p(st, u64p),
                         C.byref(wall), C.byref(lanes))
    if rc:
        raise RuntimeError(f"ref_run_local failed with status {rc}")
    keys = ["dot_bytes", "lift_bytes", "msb_bytes", "or_tree_bytes",
            "dot_rounds", "lift_rounds", "msb_rounds", "or_tree_rounds"]
    stats = [{k: int(st[8 * p + i]) for i, k in enumerate(keys)} for p in range(3)]
    return dict(person_match=pm[:ngroups].copy(), row_bits=rb[:n].copy() if debug_rows else None,
                stats=stats, wall_ms=wall.value, lanes=lanes.value)


def ref_dots_reshare(backend: int, l: int, rotations: int, seeds, db: list, s: int, q: list,
                     persons: int, membership: bool = False, variant: int = MPC_LIFT):
    """Reference L1/L2 arrays (dot_hd, dot_ml, rs_hd, rs_ml) in their ring widths;
    for plain-mask dot_ml / rs_ml are empty and `ref_dots_reshare.public_ml`
    holds the public popcounts of the last call."""
    R = ref()
    n = int(lib().orc_lane_count(persons, s, rotations, 1 if membership else 0))
    outs = [np.zeros(3 * max(1, n), np.uint32) for _ in range(4)]
    pub = np.zeros(max(1, n), np.int64)
    dbb = [np.ascontiguousarray(x, np.uint8) if len(x) else np.zeros(1, np.uint8) for x in db]
    qb = [np.ascontiguousarray(x, np.uint8) for x in q]
    dbp = (u8p * 3)(*[_p(x, u8p) for x in dbb])
    qp = (u8p * 3)(*[_p(x, u8p) for x in qb])
    rc = R.ref_dots_reshare(backend, variant, l, rotations, _p(np.ascontiguousarray(seeds, np.uint8), u8p),
                            dbp, s, qp, persons, 1 if membership else 0, _p(outs[0], u32p), _p(outs[1], u32p),
                            _p(pub, C.POINTER(C.c_int64)), _p(outs[2], u32p), _p(outs[3], u32p))
    if rc:
        raise RuntimeError(f"ref_dots_reshare failed with status {rc}")
    kh, km = code_bits(variant), mask_bits(variant)
    ref_dots_reshare.public_ml = pub[:n].copy() if km == 0 else None
    w = [kh, km or 16, kh, km or 16]
    return [o[: 3 * n].reshape(3, n).astype(_width_dtype(b)) for o, b in zip(outs, w)]


def ref_write_iris_db(path: str, codes, masks, l: int):
    c = np.ascontiguousarray(codes, np.uint64)
    m = np.ascontiguousarray(masks, np.uint64)
    rc = ref().ref_write_iris_db(os.fsencode(path), l, c.shape[0], _p(c, u64p), _p(m, u64p))
    if rc:
        raise RuntimeError(f"ref_write_iris_db failed with status {rc}")


def ref_share_files(db_path: str, backend: int, variant: int, seed: int, share_paths, seed_paths):
    """The reference `irismpc share` dealer for one variant (IRSD + IRS1 files)."""
    rc = ref().ref_share_files(os.fsencode(db_path), backend, variant, seed,
                               (C.c_char_p * 3)(*[os.fsencode(p) for p in share_paths]),
                               (C.c_char_p * 3)(*[os.fsencode(p) for p in seed_paths]))
    if rc:
        raise RuntimeError(f"ref_share_files failed with status {rc}")


def ref_read_share_file(path: str):
    """read_share_file: (backend, variant, party, l, s, payload_len) or the reference's status code."""
    hdr = np.zeros(4, np.uint32)
    s = C.c_uint64(0)
    n = C.c_uint64(0)
    rc = ref().ref_read_share_file(os.fsencode(path), _p(hdr, u32p), C.byref(s), C.byref(n))
    if rc:
        return rc
    return (*[int(x) for x in hdr], int(s.value), int(n.value))


# ------------------------------------------------- plaintext checker at scale

_plain = None


def plain_lib():
    """oracle/plain_bits.c compiled on THIS machine (-O3 -march=native, OpenMP)
    into a temporary directory: the full-scale plaintext predicate (tests only)."""
    global _plain
    if _plain is None:
        import subprocess
        import tempfile
        d = tempfile.mkdtemp(prefix="plain_bits_")
        so = os.path.join(d, "libplain_bits.so")
        cc = "/usr/bin/gcc" if os.path.exists("/usr/bin/gcc") else "gcc"
        subprocess.run([cc, "-O3", "-march=native", "-fopenmp", "-fPIC", "-shared", "-o", so,
                        os.path.join(HERE, "plain_bits.c"), "-lm"], check=True)
        P = C.CDLL(so)
        P.plain_batch_bits.argtypes = [C.c_uint32, C.c_uint32, C.c_int, C.c_int, C.c_double, C.c_uint32, C.c_uint32,
                                       C.c_uint64, u64p, u64p, C.c_uint32, u64p, u64p, u8p, u8p, u64p, u8p]
        P.plain_batch_bits.restype = C.c_uint64
        _plain = P
    return _plain


def plain_batch_bits(l: int, rotations: int, variant: int, ratio: float, db_codes, db_masks, q_codes, q_masks,
                     persons: int, membership: bool = False, expect=None, want_bits: bool = True):
    """Plaintext lane bits / person bits of a batch query (tests/oracle.hpp:35-57
    over the engine.cpp:262-293 schedule).  Returns (lane_bits or None, person bits,
    mismatches vs `expect`, first mismatching lane)."""
    P = plain_lib()
    s = db_codes.shape[0]
    n = int(lib().orc_lane_count(persons, s, rotations, 1 if membership else 0))
    bits = np.zeros(max(1, n), np.uint8) if want_bits else None
    ng = 1 if membership else persons
    pers = np.zeros(max(1, ng), np.uint8)
    fb = C.c_uint64(0)
    a = int(lib().orc_match_a(ratio))
    dc = np.ascontiguousarray(db_codes if s else np.zeros((1, words(l)), np.uint64), np.uint64)
    dm = np.ascontiguousarray(db_masks if s else np.zeros((1, words(l)), np.uint64), np.uint64)
    ex = None if expect is None else np.ascontiguousarray(expect, np.uint8)
    bad = P.plain_batch_bits(l, rotations, 1 if membership else 0, 1 if variant == PLAIN_MASK else 0, ratio, a,
                             1 << 16, s, _p(dc, u64p), _p(dm, u64p), persons,
                             _p(np.ascontiguousarray(q_codes, np.uint64), u64p),
                             _p(np.ascontiguousarray(q_masks, np.uint64), u64p), _p(bits, u8p), _p(ex, u8p),
                             C.byref(fb), _p(pers, u8p))
    return (bits[:n] if want_bits else None), pers[:ng], int(bad), int(fb.value)


# ------------------------------------- the reference's equivalence grid (_ref)

def ref_equiv_instance(backend: int, variant: int, l: int, s: int, seed: int, ratio: float):
    """equiv_common.hpp:61-89 run_instance, generated and run by the reference:
    (db_codes, db_masks, q_code, q_mask, want, got, ref_row_bits)."""
    R = ref()
    R.ref_equiv_instance.argtypes = [C.c_int, C.c_int, C.c_uint32, C.c_uint64, C.c_uint64, C.c_double, u64p, u64p,
                                     u64p, u64p, u8p, u8p, u8p]
    wl = words(l)
    dc = np.zeros((max(1, s), wl), np.uint64)
    dm = np.zeros((max(1, s), wl), np.uint64)
    qc = np.zeros(wl, np.uint64)
    qm = np.zeros(wl, np.uint64)
    want, got = C.c_uint8(0), C.c_uint8(0)
    rb = np.zeros(max(1, s), np.uint8)
    rc = R.ref_equiv_instance(backend, variant, l, s, seed, ratio, _p(dc, u64p), _p(dm, u64p), _p(qc, u64p),
                              _p(qm, u64p), C.byref(want), C.byref(got), _p(rb, u8p))
    if rc:
        raise RuntimeError(f"ref_equiv_instance failed with status {rc}")
    return dc[:s], dm[:s], qc, qm, int(want.value), int(got.value), rb[:s]


def ref_boundary_instances(count: int):
    """equiv_common.hpp:93-128 run_boundary_instances (l = 64, one DB row each)."""
    R = ref()
    R.ref_boundary_instances.argtypes = [C.c_uint, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_double),
                                         u64p, u64p, u64p, u64p, u64p, u8p, u8p]
    be = np.zeros(count, np.int32)
    va = np.zeros(count, np.int32)
    ra = np.zeros(count, np.float64)
    ms = np.zeros(count, np.uint64)
    arrs = [np.zeros(count, np.uint64) for _ in range(4)]
    want = np.zeros(count, np.uint8)
    got = np.zeros(count, np.uint8)
    rc = R.ref_boundary_instances(count, be.ctypes.data_as(C.POINTER(C.c_int)), va.ctypes.data_as(C.POINTER(C.c_int)),
                                  ra.ctypes.data_as(C.POINTER(C.c_double)), _p(ms, u64p),
                                  *[_p(a, u64p) for a in arrs], _p(want, u8p), _p(got, u8p))
    if rc:
        raise RuntimeError(f"ref_boundary_instances failed with status {rc}")
    return dict(backend=be, variant=va, ratio=ra, seed=ms, row_code=arrs[0], row_mask=arrs[1], q_code=arrs[2],
                q_mask=arrs[3], want=want, got=got)


def ref_engine_case(which: int, backend: int, variant: int):
    """test_engine.cpp:42-82: 0 planted self-match, 1 complement row, 2 ml = 0 rows."""
    R = ref()
    R.ref_engine_case.argtypes = [C.c_int, C.c_int, C.c_int, u64p, u64p, u64p, u64p, u64p, u8p, u8p]
    dc = np.zeros(8, np.uint64)
    dm = np.zeros(8, np.uint64)
    s = C.c_uint64(0)
    qc = np.zeros(1, np.uint64)
    qm = np.zeros(1, np.uint64)
    want, got = C.c_uint8(0), C.c_uint8(0)
    rc = R.ref_engine_case(which, backend, variant, _p(dc, u64p), _p(dm, u64p), C.byref(s), _p(qc, u64p),
                           _p(qm, u64p), C.byref(want), C.byref(got))
    if rc:
        raise RuntimeError(f"ref_engine_case failed with status {rc}")
    n = int(s.value)
    return dc[:n].reshape(n, 1), dm[:n].reshape(n, 1), qc, qm, int(want.value), int(got.value)


# ------------------------------------------------ comparison phase (_ref)

def synth_lanes(n: int, l: int, seed: int):
    """acceptance.cpp:48-58 synth_lanes / irismpc_cli.cpp:382-388: ml = below(l+1),
    hd = below(ml+1), dot = ml - 2 hd, from Rng(seed)."""
    rng = Rng(seed)
    dots = np.zeros(n, np.int64)
    mls = np.zeros(n, np.int64)
    for i in range(n):
        ml = rng.below(l + 1)
        hd = rng.below(ml + 1)
        mls[i] = ml
        dots[i] = ml - 2 * hd
    return dots, mls


def ref_comparison_local(variant: int, dots, mls, with_or: bool, seed: int):
    R = ref()
    R.ref_comparison_local.argtypes = [C.c_int, C.c_uint64, C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.c_int,
                                       C.c_uint64, u8p, u64p, C.POINTER(C.c_double)]
    d = np.ascontiguousarray(dots, np.int64)
    m = np.ascontiguousarray(mls, np.int64)
    op = C.c_uint8(0)
    led = np.zeros(12, np.uint64)
    wall = C.c_double(0)
    rc = R.ref_comparison_local(variant, d.size, d.ctypes.data_as(C.POINTER(C.c_int64)),
                                m.ctypes.data_as(C.POINTER(C.c_int64)), 1 if with_or else 0, seed, C.byref(op),
                                _p(led, u64p), C.byref(wall))
    if rc:
        raise RuntimeError(f"ref_comparison_local failed with status {rc}")
    keys = ("lift", "ot", "msb", "or_tree")
    return dict(opened=int(op.value), wall_ms=wall.value,
                ledger=[{k: int(led[4 * p + i]) for i, k in enumerate(keys)} for p in range(3)])


def ref_or_tree_local(bits, seed: int):
    R = ref()
    R.ref_or_tree_local.argtypes = [C.c_uint64, u8p, C.c_uint64, u8p, u64p, C.POINTER(C.c_double)]
    b = np.ascontiguousarray(bits, np.uint8)
    op = C.c_uint8(0)
    ob = np.zeros(3, np.uint64)
    wall = C.c_double(0)
    rc = R.ref_or_tree_local(b.size, _p(b, u8p), seed, C.byref(op), _p(ob, u64p), C.byref(wall))
    if rc:
        raise RuntimeError(f"ref_or_tree_local failed with status {rc}")
    return dict(opened=int(op.value), or_bytes=[int(x) for x in ob], wall_ms=wall.value)


def or_tree_batch(seeds: np.ndarray, lens, comps, stream_start=None):
    """The C restatement's or_tree_batch over caller-given bit sharings:
    comps [3][sum(lens)] component bits, groups = consecutive runs of lens[g]
    lanes.  Returns (agg [3][groups], stream positions after)."""
    L = lib()
    L.orc_or_tree_batch.argtypes = [u8p, u64p, C.c_uint32, u64p, u8p, C.c_uint64, u8p, u64p]
    ln = np.ascontiguousarray(lens, np.uint64)
    cm = np.ascontiguousarray(comps, np.uint8).reshape(3, -1)
    G = ln.size
    agg = np.zeros(3 * max(1, G), np.uint8)
    pos = np.zeros(3, np.uint64)
    st = None if stream_start is None else np.ascontiguousarray(stream_start, np.uint64)
    sd = np.ascontiguousarray(seeds, np.uint8)
    rc = L.orc_or_tree_batch(_p(sd, u8p), _p(st, u64p) if st is not None else None, G, _p(ln, u64p),
                             _p(cm, u8p), cm.shape[1], _p(agg, u8p), _p(pos, u64p))
    if rc:
        raise RuntimeError(f"orc_or_tree_batch failed with status {rc}")
    return agg[: 3 * G].reshape(3, G), pos


def ref_or_tree_batch_shares(lens, comps, seed: int):
    """The reference's own or_tree_batch (oracle/_ref, run_parties(seed), streams
    at 0) over the same input as or_tree_batch: agg components [3][groups]."""
    R = ref()
    R.ref_or_tree_batch_shares.argtypes = [C.c_uint32, u64p, u8p, C.c_uint64, C.c_uint64, u8p]
    ln = np.ascontiguousarray(lens, np.uint64)
    cm = np.ascontiguousarray(comps, np.uint8).reshape(3, -1)
    G = ln.size
    agg = np.zeros(3 * max(1, G), np.uint8)
    rc = R.ref_or_tree_batch_shares(G, _p(ln, u64p), _p(cm, u8p), cm.shape[1], seed, _p(agg, u8p))
    if rc:
        raise RuntimeError(f"ref_or_tree_batch_shares failed with status {rc}")
    return agg[: 3 * G].reshape(3, G)
