"""B200-native irismpc hot path: Python mirror of the reference query API.

The product is ``libirismpc_gpu.so`` (hand-written sm_100a CUDA behind the
C-ABI in ``include/irismpc_gpu.h``).  This module is a thin ctypes layer with
the reference's names and error behaviour:

* ``EngineConfig``          — irismpc::EngineConfig (engine.hpp:33-44)
* ``Session``               — Session::load_db / batch_query / membership
                              (engine.hpp:225-275), all three parties in one GPU
* ``run_batch_local`` / ``run_membership_local`` — cluster.hpp:82-87
* ``BoundsError`` / ``ConfigError`` / ``DeviceError`` / ``InconsistentShareError``
  — errors.hpp:22-50 mapped from the C-ABI status codes

There is no CPU fallback: importing works without a GPU, but every compute
call raises ``DeviceError`` unless the CUDA library loads and a B200 is present.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libirismpc_gpu.so")

REPLICATED, SHAMIR = 0, 1
PLAIN_MASK, MPC_LIFT, CONST_LIFT, NO_LIFT = 0, 1, 2, 3  # Variant (shares.hpp:28)
VARIANTS = {"plain-mask": PLAIN_MASK, "mpc-lift": MPC_LIFT, "const-lift": CONST_LIFT, "no-lift": NO_LIFT}
# (hamming dot bits, mask dot bits (0 = public mask bits), comparison bits), shares.hpp:37-48
VARIANT_WIDTHS = {PLAIN_MASK: (16, 0, 16), MPC_LIFT: (16, 16, 32), CONST_LIFT: (16, 32, 32), NO_LIFT: (32, 32, 32)}

TAP_DOT_HD, TAP_DOT_ML, TAP_RS_HD, TAP_RS_ML, TAP_ML32, TAP_DIFF, TAP_MSB, TAP_AGG = range(1, 9)

EXPORTED = [
    "irismpc_gpu_seeds_from_master", "irismpc_gpu_record_bytes", "irismpc_gpu_lane_count",
    "irismpc_gpu_create", "irismpc_gpu_destroy", "irismpc_gpu_last_error", "irismpc_gpu_stream",
    "irismpc_gpu_load_db", "irismpc_gpu_load_db_device", "irismpc_gpu_batch_query",
    "irismpc_gpu_batch_query_device", "irismpc_gpu_membership", "irismpc_gpu_batch_query_partial",
    "irismpc_gpu_or_open", "irismpc_gpu_get_stream_positions", "irismpc_gpu_set_stream_positions",
    "irismpc_gpu_synth_records", "irismpc_gpu_deal_payload", "irismpc_gpu_synth_db",
    "irismpc_gpu_enable_taps", "irismpc_gpu_read_tap", "irismpc_gpu_profile", "irismpc_gpu_profile_read",
    "irismpc_gpu_tap_rows", "irismpc_gpu_threshold_kernels", "irismpc_gpu_comparison_only", "irismpc_gpu_or_tree_only",
    "irismpc_gpu_shard_group_create", "irismpc_gpu_shard_group_destroy", "irismpc_gpu_shard_attach_inproc",
    "irismpc_gpu_shard_attach_nccl", "irismpc_gpu_sharded_batch_query", "irismpc_gpu_sharded_batch_query_device",
    "irismpc_gpu_sharded_membership", "irismpc_gpu_batch_query_submit", "irismpc_gpu_batch_query_wait",
    "irismpc_gpu_sharded_batch_query_submit",
    "irismpc_gpu_read_share_header", "irismpc_gpu_write_share_file", "irismpc_gpu_load_db_files",
    "irismpc_gpu_read_seed_files", "irismpc_gpu_write_seed_file", "irismpc_gpu_read_iris_db_header",
    "irismpc_gpu_read_iris_db", "irismpc_gpu_write_iris_db",
    "irismpc_gpu_nccl_unique_id", "irismpc_gpu_party_create_nccl", "irismpc_gpu_inproc_create",
    "irismpc_gpu_inproc_destroy", "irismpc_gpu_party_create_inproc", "irismpc_gpu_party_destroy",
    "irismpc_gpu_party_last_error", "irismpc_gpu_party_load_db", "irismpc_gpu_party_batch_query",
    "irismpc_gpu_party_membership", "irismpc_gpu_party_read_tap", "irismpc_gpu_party_stream_positions",
]


class IrisError(RuntimeError):
    code = 1


class ConfigError(IrisError):
    """irismpc::Error / ConfigMismatchError (payload size, unsupported config)."""
    code = 2


class DeviceError(IrisError):
    """TransportError analogue: CUDA failure or no B200."""
    code = 3


class BoundsError(IrisError):
    """irismpc::BoundsError (EngineConfig::validate)."""
    code = 4


class InconsistentShareError(IrisError):
    """irismpc::InconsistentShareError (replication cross-check)."""
    code = 5


_ERRORS = {c.code: c for c in (IrisError, ConfigError, DeviceError, BoundsError, InconsistentShareError)}


class _Config(C.Structure):
    _fields_ = [("backend", C.c_uint32), ("variant", C.c_uint32), ("l", C.c_uint32), ("a", C.c_uint32),
                ("b", C.c_uint32), ("m", C.c_uint32), ("rotations", C.c_uint32), ("debug_rows", C.c_uint32),
                ("seeds", C.c_uint8 * 48), ("device", C.c_int32), ("shard_rank", C.c_uint32),
                ("db_rows_total", C.c_uint64), ("db_row_offset", C.c_uint64), ("match_ratio", C.c_double),
                ("reserved", C.c_uint64 * 3)]


class ShareHeader(C.Structure):
    """ShareFileHeader (io.hpp:38-47)."""
    _fields_ = [("backend", C.c_uint32), ("variant", C.c_uint32), ("party", C.c_uint32), ("l", C.c_uint32),
                ("s", C.c_uint64)]


class PartyStats(C.Structure):
    """One party's QueryStats from the measured ledger (party mode)."""
    _fields_ = [(k, C.c_uint64) for k in ("s", "l", "batch", "lanes", "dot_bytes", "lift_bytes", "msb_bytes",
                                          "or_tree_bytes", "dot_rounds", "lift_rounds", "msb_rounds",
                                          "or_tree_rounds", "wire_bytes")] + [("wall_ms", C.c_double),
                                                                                ("phase_ms", C.c_double * 6)]

    def ledger(self) -> dict:
        return {k: getattr(self, k) for k in ("dot_bytes", "lift_bytes", "msb_bytes", "or_tree_bytes", "dot_rounds",
                                              "lift_rounds", "msb_rounds", "or_tree_rounds")}


class Stats(C.Structure):
    """QueryStats (engine.hpp:46-56) per party + device phase times."""
    _fields_ = [("s", C.c_uint64), ("l", C.c_uint64), ("batch", C.c_uint64), ("lanes", C.c_uint64),
                ("dot_bytes", C.c_uint64 * 3), ("lift_bytes", C.c_uint64 * 3), ("msb_bytes", C.c_uint64 * 3),
                ("or_tree_bytes", C.c_uint64 * 3), ("dot_rounds", C.c_uint64), ("lift_rounds", C.c_uint64),
                ("msb_rounds", C.c_uint64), ("or_tree_rounds", C.c_uint64), ("wall_ms", C.c_double),
                ("prep_ms", C.c_double), ("gemm_ms", C.c_double), ("threshold_ms", C.c_double),
                ("or_ms", C.c_double), ("gemm_launches", C.c_uint64), ("kernel_launches", C.c_uint64),
                ("gemm_int8_ops", C.c_uint64), ("rotation_pair_gemm", C.c_uint32)]

    def party(self, p: int) -> dict:
        return dict(dot_bytes=self.dot_bytes[p], lift_bytes=self.lift_bytes[p], msb_bytes=self.msb_bytes[p],
                    or_tree_bytes=self.or_tree_bytes[p], dot_rounds=self.dot_rounds,
                    lift_rounds=self.lift_rounds, msb_rounds=self.msb_rounds, or_tree_rounds=self.or_tree_rounds)


_lib = None
vp = C.c_void_p
u8p = C.POINTER(C.c_uint8)
u64p = C.POINTER(C.c_uint64)
szp = C.POINTER(C.c_size_t)


def lib() -> C.CDLL:
    """Loads the CUDA library; raises DeviceError if it is missing (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise DeviceError(f"{LIB_PATH} is missing: run `python -m paper_2405_04463_b200.build` "
                              "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        L.irismpc_gpu_seeds_from_master.argtypes = [C.c_uint64, u8p]
        L.irismpc_gpu_record_bytes.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32]
        L.irismpc_gpu_record_bytes.restype = C.c_size_t
        L.irismpc_gpu_lane_count.argtypes = [C.c_uint32, C.c_uint64, C.c_uint32, C.c_int]
        L.irismpc_gpu_lane_count.restype = C.c_uint64
        L.irismpc_gpu_create.argtypes = [C.POINTER(_Config), C.POINTER(vp)]
        L.irismpc_gpu_destroy.argtypes = [vp]
        L.irismpc_gpu_last_error.argtypes = [vp]
        L.irismpc_gpu_last_error.restype = C.c_char_p
        L.irismpc_gpu_stream.argtypes = [vp]
        L.irismpc_gpu_stream.restype = vp
        P3 = vp * 3
        S3 = C.c_size_t * 3
        for f in ("irismpc_gpu_load_db", "irismpc_gpu_load_db_device"):
            getattr(L, f).argtypes = [vp, P3, S3, C.c_uint64]
        for f in ("irismpc_gpu_batch_query", "irismpc_gpu_batch_query_device"):
            getattr(L, f).argtypes = [vp, P3, S3, C.c_uint32, vp, vp, C.POINTER(Stats)]
        L.irismpc_gpu_membership.argtypes = [vp, P3, S3, vp, vp, C.POINTER(Stats)]
        L.irismpc_gpu_batch_query_partial.argtypes = [vp, P3, S3, C.c_uint32, vp, C.POINTER(Stats)]
        L.irismpc_gpu_or_open.argtypes = [vp, vp, C.c_uint32, C.c_uint32, vp]
        L.irismpc_gpu_get_stream_positions.argtypes = [vp, u64p]
        L.irismpc_gpu_set_stream_positions.argtypes = [vp, u64p]
        L.irismpc_gpu_synth_records.argtypes = [vp, C.c_uint64, C.c_uint64, C.c_uint64, C.c_double, vp, vp]
        L.irismpc_gpu_deal_payload.argtypes = [vp, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, vp, vp, P3]
        L.irismpc_gpu_synth_db.argtypes = [vp, C.c_uint64, C.c_uint64, C.c_uint64, C.c_double, C.c_uint64]
        L.irismpc_gpu_enable_taps.argtypes = [vp, C.c_int]
        L.irismpc_gpu_profile.argtypes = [vp, C.c_int]
        L.irismpc_gpu_tap_rows.argtypes = [vp, u64p, C.c_uint32]
        L.irismpc_gpu_threshold_kernels.argtypes = [vp, C.c_int]
        L.irismpc_gpu_comparison_only.argtypes = [vp, P3, S3, P3, S3, C.c_uint64, C.c_int, vp, vp, C.POINTER(Stats)]
        L.irismpc_gpu_or_tree_only.argtypes = [vp, P3, S3, C.c_uint64, vp, C.POINTER(Stats)]
        L.irismpc_gpu_shard_group_create.argtypes = [C.c_uint32, C.POINTER(vp)]
        L.irismpc_gpu_shard_group_destroy.argtypes = [vp]
        L.irismpc_gpu_shard_attach_inproc.argtypes = [vp, vp]
        L.irismpc_gpu_shard_attach_nccl.argtypes = [vp, u8p, C.c_uint32]
        for f in ("irismpc_gpu_sharded_batch_query", "irismpc_gpu_sharded_batch_query_device"):
            getattr(L, f).argtypes = [vp, P3, S3, C.c_uint32, vp, C.POINTER(Stats)]
        L.irismpc_gpu_sharded_membership.argtypes = [vp, P3, S3, vp, C.POINTER(Stats)]
        L.irismpc_gpu_batch_query_submit.argtypes = [vp, P3, S3, C.c_uint32, vp, C.POINTER(C.c_uint64)]
        L.irismpc_gpu_batch_query_wait.argtypes = [vp, C.c_uint64, C.POINTER(Stats)]
        L.irismpc_gpu_sharded_batch_query_submit.argtypes = [vp, P3, S3, C.c_uint32, vp, C.POINTER(C.c_uint64)]
        L.irismpc_gpu_profile_read.argtypes = [vp, vp, vp, vp, C.c_uint32, C.POINTER(C.c_uint32)]
        L.irismpc_gpu_read_tap.argtypes = [vp, C.c_int, vp, C.c_size_t]
        cp3 = C.c_char_p * 3
        L.irismpc_gpu_read_share_header.argtypes = [C.c_char_p, C.POINTER(ShareHeader)]
        L.irismpc_gpu_write_share_file.argtypes = [C.c_char_p, C.POINTER(ShareHeader), vp, C.c_size_t]
        L.irismpc_gpu_load_db_files.argtypes = [vp, cp3]
        L.irismpc_gpu_read_seed_files.argtypes = [cp3, u8p]
        L.irismpc_gpu_write_seed_file.argtypes = [C.c_char_p, C.c_uint32, u8p, u8p]
        L.irismpc_gpu_read_iris_db_header.argtypes = [C.c_char_p, C.POINTER(C.c_uint32), C.POINTER(C.c_uint64)]
        L.irismpc_gpu_read_iris_db.argtypes = [C.c_char_p, vp, vp, C.c_uint64]
        L.irismpc_gpu_write_iris_db.argtypes = [C.c_char_p, C.c_uint32, C.c_uint64, vp, vp]
        L.irismpc_gpu_nccl_unique_id.argtypes = [u8p]
        L.irismpc_gpu_party_create_nccl.argtypes = [C.POINTER(_Config), C.c_uint32, u8p, C.POINTER(vp)]
        L.irismpc_gpu_inproc_create.argtypes = [C.POINTER(vp)]
        L.irismpc_gpu_inproc_destroy.argtypes = [vp]
        L.irismpc_gpu_party_create_inproc.argtypes = [C.POINTER(_Config), C.c_uint32, vp, C.POINTER(vp)]
        L.irismpc_gpu_party_destroy.argtypes = [vp]
        L.irismpc_gpu_party_last_error.argtypes = [vp]
        L.irismpc_gpu_party_last_error.restype = C.c_char_p
        L.irismpc_gpu_party_load_db.argtypes = [vp, vp, C.c_size_t, C.c_uint64]
        L.irismpc_gpu_party_batch_query.argtypes = [vp, vp, C.c_size_t, C.c_uint32, vp, vp, C.POINTER(PartyStats)]
        L.irismpc_gpu_party_membership.argtypes = [vp, vp, C.c_size_t, vp, vp, C.POINTER(PartyStats)]
        L.irismpc_gpu_party_read_tap.argtypes = [vp, C.c_int, vp, C.c_size_t]
        L.irismpc_gpu_party_stream_positions.argtypes = [vp, u64p]
        _lib = L
    return _lib


def seeds_from_master(seed: int) -> np.ndarray:
    out = np.zeros(48, np.uint8)
    lib().irismpc_gpu_seeds_from_master(seed, out.ctypes.data_as(u8p))
    return out


def record_bytes(backend: int, l: int, variant: int = MPC_LIFT) -> int:
    """code_record_bytes + mask_record_bytes (shares.cpp:49-59)."""
    return int(lib().irismpc_gpu_record_bytes(backend, variant, l))


# ---- files (io.hpp:28-60) -------------------------------------------------------

def _b(path) -> bytes:
    return os.fsencode(path)


def read_share_header(path) -> ShareHeader:
    """read_share_file's header and size checks; raises ConfigError like the reference's Error."""
    h = ShareHeader()
    if lib().irismpc_gpu_read_share_header(_b(path), C.byref(h)):
        raise ConfigError(f"not a valid IRS1 share file: {path}")
    return h


def write_share_file(path, backend: int, variant: int, party: int, l: int, s: int, payload) -> None:
    h = ShareHeader(backend, variant, party, l, s)
    buf = np.ascontiguousarray(np.frombuffer(payload, np.uint8) if isinstance(payload, (bytes, bytearray))
                               else payload, np.uint8)
    if lib().irismpc_gpu_write_share_file(_b(path), C.byref(h), buf.ctypes.data, buf.nbytes):
        raise ConfigError(f"cannot write {path}")


def read_seed_files(paths) -> np.ndarray:
    """Three IRSD files (parties 1..3) -> seed_1 | seed_2 | seed_3, cross-checked."""
    out = np.zeros(48, np.uint8)
    if lib().irismpc_gpu_read_seed_files((C.c_char_p * 3)(*[_b(p) for p in paths]), out.ctypes.data_as(u8p)):
        raise ConfigError("bad or inconsistent IRSD seed files")
    return out


def write_seed_file(path, party: int, own, prev) -> None:
    o = np.ascontiguousarray(own, np.uint8)
    p = np.ascontiguousarray(prev, np.uint8)
    if lib().irismpc_gpu_write_seed_file(_b(path), party, o.ctypes.data_as(u8p), p.ctypes.data_as(u8p)):
        raise ConfigError(f"cannot write {path}")


def read_iris_db(path):
    """IRMP plaintext DB -> (codes, masks) uint64 word arrays [s][(l+63)/64], and l."""
    l, s = C.c_uint32(0), C.c_uint64(0)
    if lib().irismpc_gpu_read_iris_db_header(_b(path), C.byref(l), C.byref(s)):
        raise ConfigError(f"not a valid IRMP file: {path}")
    wl = (l.value + 63) // 64
    codes = np.zeros((max(1, s.value), wl), np.uint64)
    masks = np.zeros((max(1, s.value), wl), np.uint64)
    if lib().irismpc_gpu_read_iris_db(_b(path), codes.ctypes.data, masks.ctypes.data, s.value):
        raise ConfigError(f"cannot read {path}")
    return codes[: s.value], masks[: s.value], l.value


def write_iris_db(path, codes: np.ndarray, masks: np.ndarray, l: int) -> None:
    c = np.ascontiguousarray(codes, np.uint64)
    m = np.ascontiguousarray(masks, np.uint64)
    if lib().irismpc_gpu_write_iris_db(_b(path), l, c.shape[0], c.ctypes.data, m.ctypes.data):
        raise ConfigError(f"cannot write {path}")


def lane_count(persons: int, s: int, rotations: int, membership: bool = False) -> int:
    return int(lib().irismpc_gpu_lane_count(persons, s, rotations, 1 if membership else 0))


def match_a(ratio: float) -> int:
    """MatchParams::make(ratio, 16).a (iris.hpp:163-174)."""
    b = 1 << 16
    x = (1.0 - 2.0 * ratio) * b  # llround: halves away from zero
    a = int(np.floor(x + 0.5)) if x >= 0 else -int(np.floor(-x + 0.5))
    return min(a, b)


@dataclass
class EngineConfig:
    """irismpc::EngineConfig (engine.hpp:33-44); variant defaults to mpc-lift."""
    backend: int = SHAMIR
    l: int = 12800
    match_ratio: float = 0.375
    rotations: int = 31
    debug_rows: bool = False
    variant: int = MPC_LIFT
    m: int = 16
    a: int | None = None
    b: int = 1 << 16

    def params(self) -> tuple[int, int]:
        return (self.a if self.a is not None else match_a(self.match_ratio)), self.b


def _ptr(x) -> int:
    """Data pointer of a numpy array or torch tensor."""
    if hasattr(x, "data_ptr"):
        return int(x.data_ptr())
    return int(x.ctypes.data)


def _nbytes(x) -> int:
    if hasattr(x, "element_size"):
        return int(x.numel() * x.element_size())
    return int(x.nbytes)


class Session:
    """All three parties of one DB shard on one GPU (Session<B,16,16>)."""

    def __init__(self, cfg: EngineConfig, seeds: np.ndarray | None = None, master_seed: int | None = None,
                 device: int = 0, shard_rank: int = 0, db_rows_total: int = 0, db_row_offset: int = 0):
        L = lib()
        self.cfg = cfg
        a, b = cfg.params()
        c = _Config()
        c.backend, c.variant, c.l, c.a, c.b, c.m = cfg.backend, cfg.variant, cfg.l, a, b, cfg.m
        c.rotations, c.debug_rows = cfg.rotations, 1 if cfg.debug_rows else 0
        c.match_ratio = cfg.match_ratio
        if seeds is None:
            seeds = seeds_from_master(master_seed if master_seed is not None else 0)
        for i in range(48):
            c.seeds[i] = int(seeds[i])
        c.device, c.shard_rank, c.db_rows_total, c.db_row_offset = device, shard_rank, db_rows_total, db_row_offset
        h = vp()
        rc = L.irismpc_gpu_create(C.byref(c), C.byref(h))
        if rc:
            raise _ERRORS.get(rc, IrisError)(f"irismpc_gpu_create failed ({rc})")
        self._h = h
        self.s = 0
        self.rec = record_bytes(cfg.backend, cfg.l, cfg.variant)
        self.last_stats = Stats()

    def close(self):
        if getattr(self, "_h", None):
            lib().irismpc_gpu_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def _check(self, rc: int):
        if rc:
            msg = lib().irismpc_gpu_last_error(self._h).decode()
            raise _ERRORS.get(rc, IrisError)(msg)

    @property
    def stream(self) -> int:
        return int(lib().irismpc_gpu_stream(self._h) or 0)

    # -- DB ---------------------------------------------------------------
    def load_db(self, payloads, s: int):
        """Session::load_db: three host payloads (bytes/np.uint8) or device tensors."""
        dev = hasattr(payloads[0], "is_cuda") and payloads[0].is_cuda
        arrs = [p if hasattr(p, "data_ptr") else np.ascontiguousarray(np.frombuffer(p, np.uint8) if isinstance(p, (bytes, bytearray)) else p)
                for p in payloads]
        ptrs = (vp * 3)(*[_ptr(a) for a in arrs])
        lens = (C.c_size_t * 3)(*[_nbytes(a) for a in arrs])
        f = lib().irismpc_gpu_load_db_device if dev else lib().irismpc_gpu_load_db
        self._check(f(self._h, ptrs, lens, s))
        self.s = s

    def load_db_files(self, paths):
        """Session::load_db from the parties' IRS1 share files (streamed into HBM)."""
        h = read_share_header(paths[0])
        self._check(lib().irismpc_gpu_load_db_files(self._h, (C.c_char_p * 3)(*[_b(p) for p in paths])))
        self.s = int(h.s)

    def synth_db(self, s: int, rng_seed: int = 2, first: int = 0, mask_density: float = 0.9, deal_seed: int = 7):
        """Device dealer: rows [first, first+s) of Rng(rng_seed) random_record, dealt with sub_rng(deal_seed,1)."""
        self._check(lib().irismpc_gpu_synth_db(self._h, s, rng_seed, first, mask_density, deal_seed))
        self.s = s

    def synth_records(self, rng_seed: int, first: int, count: int, mask_density: float, codes, masks):
        self._check(lib().irismpc_gpu_synth_records(self._h, rng_seed, first, count, mask_density,
                                                    _ptr(codes), _ptr(masks)))

    def deal_payload(self, deal_seed: int, tag: int, first_record: int, codes, masks, outs):
        nrec = codes.shape[0]
        ptrs = (vp * 3)(*[_ptr(o) for o in outs])
        self._check(lib().irismpc_gpu_deal_payload(self._h, deal_seed, tag, first_record, nrec, _ptr(codes),
                                                   _ptr(masks), ptrs))

    # -- queries ------------------------------------------------------------
    def _q(self, q):
        dev = hasattr(q[0], "is_cuda") and q[0].is_cuda
        arrs = [x if hasattr(x, "data_ptr") else np.ascontiguousarray(x, np.uint8) for x in q]
        return dev, arrs, (vp * 3)(*[_ptr(a) for a in arrs]), (C.c_size_t * 3)(*[_nbytes(a) for a in arrs])

    def batch_query(self, q, persons: int, want_rows: bool = False) -> np.ndarray:
        """Session::batch_query: q = three payloads of 2*persons codes; returns person_match at P1."""
        dev, arrs, ptrs, lens = self._q(q)
        out = np.zeros(max(1, persons), np.uint8)
        rows = np.zeros(max(1, lane_count(persons, self.s, self.cfg.rotations)), np.uint8) if want_rows else None
        f = lib().irismpc_gpu_batch_query_device if dev else lib().irismpc_gpu_batch_query
        self._check(f(self._h, ptrs, lens, persons, out.ctypes.data, rows.ctypes.data if want_rows else None,
                      C.byref(self.last_stats)))
        self.row_bits = rows
        return out[:persons]

    def batch_query_submit(self, q, persons: int) -> int:
        """Streaming batch query (device payloads kept alive until the wait): returns a ticket."""
        dev, arrs, ptrs, lens = self._q(q)
        if not dev:
            raise ConfigError("batch_query_submit expects device-resident payloads")
        out = np.zeros(max(1, persons), np.uint8)
        t = C.c_uint64(0)
        self._check(lib().irismpc_gpu_batch_query_submit(self._h, ptrs, lens, persons, out.ctypes.data, C.byref(t)))
        if not hasattr(self, "_inflight"):
            self._inflight = {}
        self._inflight[t.value] = (out[:persons], arrs)
        return t.value

    def batch_query_wait(self, ticket: int) -> np.ndarray:
        """Completes a streaming query: its person_match (stats in last_stats)."""
        self._check(lib().irismpc_gpu_batch_query_wait(self._h, ticket, C.byref(self.last_stats)))
        out, _ = self._inflight.pop(ticket)
        return out

    def membership(self, q, want_rows: bool = False) -> bool:
        """Session::membership: one code, no rotation."""
        dev, arrs, ptrs, lens = self._q(q)
        if dev:
            arrs = [a.cpu().numpy() for a in arrs]
            ptrs = (vp * 3)(*[_ptr(a) for a in arrs])
        out = np.zeros(1, np.uint8)
        rows = np.zeros(max(1, self.s), np.uint8) if want_rows else None
        self._check(lib().irismpc_gpu_membership(self._h, ptrs, lens, out.ctypes.data,
                                                 rows.ctypes.data if want_rows else None,
                                                 C.byref(self.last_stats)))
        self.row_bits = rows
        return bool(out[0])

    def batch_query_partial(self, q, persons: int, partial_out):
        """Shard query up to the per-person shared aggregate (device [3][persons] bytes, unopened)."""
        dev, arrs, ptrs, lens = self._q(q)
        if not dev:
            raise ConfigError("batch_query_partial expects device-resident payloads")
        self._check(lib().irismpc_gpu_batch_query_partial(self._h, ptrs, lens, persons, _ptr(partial_out),
                                                          C.byref(self.last_stats)))

    def or_open(self, partials, G: int, persons: int) -> np.ndarray:
        out = np.zeros(max(1, persons), np.uint8)
        self._check(lib().irismpc_gpu_or_open(self._h, _ptr(partials), G, persons, out.ctypes.data))
        return out[:persons]

    # -- DB-sharded queries (one context per shard) ------------------
    def shard_attach_inproc(self, group: "ShardGroup"):
        """Join an in-process shard group (several contexts in one process)."""
        self._check(lib().irismpc_gpu_shard_attach_inproc(self._h, group._h))
        self._group = group

    def shard_attach_nccl(self, nccl_id: bytes, world: int):
        """Join the NCCL communicator of `world` shards (rank = this context's shard_rank)."""
        idb = np.frombuffer(nccl_id, np.uint8).copy()
        self._check(lib().irismpc_gpu_shard_attach_nccl(self._h, idb.ctypes.data_as(u8p), world))

    def sharded_batch_query(self, q, persons: int, qlen=None) -> np.ndarray | None:
        """Broadcast (from shard 0) -> shard query -> gather -> MPC-OR + open on shard 0.
        q: three payloads (host arrays or device tensors) on shard 0, None elsewhere
        (then qlen gives the payload sizes).  Returns person_match on shard 0."""
        if q is not None:
            dev, arrs, ptrs, lens = self._q(q)
        else:
            dev, ptrs, lens = True, (vp * 3)(None, None, None), (C.c_size_t * 3)(*qlen)
        out = np.zeros(max(1, persons), np.uint8)
        f = lib().irismpc_gpu_sharded_batch_query_device if dev else lib().irismpc_gpu_sharded_batch_query
        self._check(f(self._h, ptrs, lens, persons, out.ctypes.data, C.byref(self.last_stats)))
        return out[:persons]

    def sharded_batch_query_submit(self, q, persons: int, qlen=None) -> int:
        """Streaming sharded query (NCCL attach): device payloads on shard 0 (None elsewhere,
        qlen then gives their sizes); complete with batch_query_wait (person_match on shard 0)."""
        if q is not None:
            dev, arrs, ptrs, lens = self._q(q)
            if not dev:
                raise ConfigError("sharded_batch_query_submit expects device-resident payloads")
        else:
            arrs, ptrs, lens = None, (vp * 3)(None, None, None), (C.c_size_t * 3)(*qlen)
        out = np.zeros(max(1, persons), np.uint8)
        t = C.c_uint64(0)
        self._check(lib().irismpc_gpu_sharded_batch_query_submit(self._h, ptrs, lens, persons, out.ctypes.data,
                                                                 C.byref(t)))
        if not hasattr(self, "_inflight"):
            self._inflight = {}
        self._inflight[t.value] = (out[:persons], arrs)
        return t.value

    # -- the comparison phase alone ---------------------------------------------
    def comparison_only(self, hd_payloads, ml_payloads, lanes: int, with_or_tree: bool = False,
                        want_bits: bool = False):
        """party_comparison_only for all three parties (engine.cpp:448-515): returns
        (opened aggregate or None, opened per-lane MSB bits or None)."""
        hp = [np.ascontiguousarray(x, np.uint8) for x in hd_payloads]
        mp = [np.ascontiguousarray(x, np.uint8) for x in ml_payloads]
        op = np.zeros(1, np.uint8)
        bits = np.zeros(max(1, lanes), np.uint8) if want_bits else None
        self._check(lib().irismpc_gpu_comparison_only(
            self._h, (vp * 3)(*[a.ctypes.data for a in hp]), (C.c_size_t * 3)(*[a.nbytes for a in hp]),
            (vp * 3)(*[a.ctypes.data for a in mp]), (C.c_size_t * 3)(*[a.nbytes for a in mp]), lanes,
            1 if with_or_tree else 0, op.ctypes.data, bits.ctypes.data if want_bits else None,
            C.byref(self.last_stats)))
        return (int(op[0]) if with_or_tree else None), (bits[:lanes] if want_bits else None)

    def or_tree_only(self, payloads, lanes: int) -> int:
        """party_or_tree_only for all three parties (engine.cpp:517-532): the opened OR."""
        pp = [np.ascontiguousarray(x, np.uint8) for x in payloads]
        op = np.zeros(1, np.uint8)
        self._check(lib().irismpc_gpu_or_tree_only(self._h, (vp * 3)(*[a.ctypes.data for a in pp]),
                                                   (C.c_size_t * 3)(*[a.nbytes for a in pp]), lanes,
                                                   op.ctypes.data, C.byref(self.last_stats)))
        return int(op[0])

    # -- streams / taps --------------------------------------------------------
    def stream_positions(self) -> np.ndarray:
        p = np.zeros(3, np.uint64)
        self._check(lib().irismpc_gpu_get_stream_positions(self._h, p.ctypes.data_as(u64p)))
        return p

    def set_stream_positions(self, pos):
        p = np.ascontiguousarray(pos, np.uint64)
        self._check(lib().irismpc_gpu_set_stream_positions(self._h, p.ctypes.data_as(u64p)))

    def profile(self, on: bool = True):
        """Serialised queries with per-kernel CUDA events (irismpc_gpu_profile)."""
        self._check(lib().irismpc_gpu_profile(self._h, 1 if on else 0))

    def threshold_kernels(self, tile: bool):
        """irismpc_gpu_threshold_kernels: tile (True) or lane-major (False, default) reshare / inject."""
        self._check(lib().irismpc_gpu_threshold_kernels(self._h, 1 if tile else 0))

    def profile_read(self) -> dict:
        """{kernel name: (device ms, launches)} accumulated since the last read."""
        mx = 64
        names = (C.c_char * (48 * mx))()
        ms = np.zeros(mx, np.float64)
        cnt = np.zeros(mx, np.uint64)
        n = C.c_uint32(0)
        self._check(lib().irismpc_gpu_profile_read(self._h, names, ms.ctypes.data, cnt.ctypes.data, mx, C.byref(n)))
        raw = bytes(names)
        return {raw[48 * i:48 * i + 48].split(b"\0")[0].decode(): (float(ms[i]), int(cnt[i])) for i in range(n.value)}

    def tap_rows(self, rows) -> None:
        """Row-sampled L1 taps (irismpc_gpu_tap_rows); [] turns them off."""
        r = np.ascontiguousarray(rows, np.uint64)
        self._check(lib().irismpc_gpu_tap_rows(self._h, r.ctypes.data_as(u64p) if r.size else None, r.size))
        self._tap_k = int(r.size)

    def read_row_taps(self, tap: int, persons: int) -> np.ndarray:
        """[3][ncols * k + pairs] (plain-mask DOT_ML: [ncols * k + pairs]) of the last query."""
        n = 2 * persons * self.cfg.rotations * self._tap_k + persons * (persons - 1) // 2 * 4 * self.cfg.rotations
        return self.read_tap(tap, n)

    def enable_taps(self, on: bool = True):
        self._check(lib().irismpc_gpu_enable_taps(self._h, 1 if on else 0))

    def read_tap(self, tap: int, n: int) -> np.ndarray:
        """Tap arrays [3][n] (plain-mask TAP_DOT_ML: [n] public popcounts), in the
        ring's width: u16 for 16-bit dots and reshared 16-bit shares, else u32."""
        kh, km, kc = VARIANT_WIDTHS[self.cfg.variant]
        rows = 1 if (tap == TAP_DOT_ML and km == 0) else 3
        dt = {TAP_DOT_HD: np.uint16 if kh == 16 else np.uint32,
              TAP_DOT_ML: np.uint32 if km == 32 else np.uint16,
              TAP_MSB: np.uint8, TAP_AGG: np.uint8}.get(tap, np.uint32)
        out = np.zeros(rows * n, dt)
        self._check(lib().irismpc_gpu_read_tap(self._h, tap, out.ctypes.data, out.nbytes))
        out = out.reshape(rows, n)
        if rows == 1:
            return out[0]
        if (tap == TAP_RS_HD and kh == 16) or (tap == TAP_RS_ML and km == 16):
            return out.astype(np.uint16)
        if tap == TAP_DIFF and kc == 16:
            return out.astype(np.uint16)
        return out


class ShardGroup:
    """In-process group of DB shards (irismpc_gpu_shard_group): the query broadcast
    and partial gather between contexts of one process, one host thread each."""

    def __init__(self, world: int):
        h = vp()
        if lib().irismpc_gpu_shard_group_create(world, C.byref(h)):
            raise ConfigError("shard group")
        self._h, self.world = h, world

    def close(self):
        if getattr(self, "_h", None):
            lib().irismpc_gpu_shard_group_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def share_lane_values(values, bits: int, rng: np.random.Generator):
    """Replicated 3-party shares of signed per-lane values in Z_2^bits as the
    three parties' bench payloads: party p holds (own = x_p, prev = x_{p-1}),
    little-endian (emit_rep_share_list, src/cluster.cpp:83-95; any uniformly
    random sharing -- the opened outputs do not depend on it)."""
    v = np.asarray(values, np.int64)
    mod = 1 << bits
    dt = np.uint16 if bits == 16 else np.uint32
    x1 = rng.integers(0, mod, v.size, dtype=np.uint64)
    x2 = rng.integers(0, mod, v.size, dtype=np.uint64)
    x3 = (v.astype(np.uint64) - x1 - x2) % np.uint64(mod)
    xs = [x1.astype(dt), x2.astype(dt), x3.astype(dt)]
    out = []
    for p in range(3):
        pair = np.empty((v.size, 2), dt)
        pair[:, 0] = xs[p]
        pair[:, 1] = xs[(p + 2) % 3]
        out.append(pair.view(np.uint8).ravel())
    return out


def share_bit_words(bits, rng: np.random.Generator):
    """Replicated XOR shares of a lane bit vector as party payloads of
    (own u64, prev u64) per 64-lane word (run_or_tree_local, cluster.cpp:147-165)."""
    b = np.asarray(bits, np.uint8)
    W = (b.size + 63) // 64
    padded = np.zeros(64 * W, np.uint8)
    padded[:b.size] = b
    plain = np.packbits(padded, bitorder="little").view(np.uint64)
    x1 = rng.integers(0, 2**63, W, dtype=np.uint64) ^ (rng.integers(0, 2, W, dtype=np.uint64) << np.uint64(63))
    x2 = rng.integers(0, 2**63, W, dtype=np.uint64) ^ (rng.integers(0, 2, W, dtype=np.uint64) << np.uint64(63))
    x3 = plain ^ x1 ^ x2
    xs = [x1, x2, x3]
    return [np.stack([xs[p], xs[(p + 2) % 3]], 1).view(np.uint8).ravel() for p in range(3)]


def _dealt_on_device(sess: Session, codes: np.ndarray, masks: np.ndarray, seed: int, tag: int):
    import torch
    dc = torch.from_numpy(np.ascontiguousarray(codes).view(np.int64)).cuda()
    dm = torch.from_numpy(np.ascontiguousarray(masks).view(np.int64)).cuda()
    n = codes.shape[0]
    outs = [torch.empty(max(1, n * sess.rec), dtype=torch.uint8, device="cuda") for _ in range(3)]
    if n:
        sess.deal_payload(seed, tag, 0, dc, dm, outs)
    return [o[: n * sess.rec] for o in outs]


def run_batch_local(cfg: EngineConfig, q_codes: np.ndarray, q_masks: np.ndarray, db_codes: np.ndarray,
                    db_masks: np.ndarray, seed: int, persons: int | None = None, membership: bool = False,
                    want_rows: bool = False, taps: bool = False, device: int = 0):
    """run_batch_local / run_membership_local (cluster.cpp:30-79) on one B200.

    Deals the DB with sub_rng(seed,1) and the queries with sub_rng(seed,2) on the
    device (bit-identical payloads to the reference dealer), party seeds from
    `seed`.  Returns (person_match, session)."""
    sess = Session(cfg, master_seed=seed, device=device)
    s = db_codes.shape[0]
    db = _dealt_on_device(sess, db_codes, db_masks, seed, 1)
    sess.load_db(db, s)
    q = _dealt_on_device(sess, q_codes, q_masks, seed, 2)
    if taps:
        sess.enable_taps(True)
    if membership:
        m = np.array([sess.membership(q, want_rows)], np.uint8)
    else:
        m = sess.batch_query(q, persons if persons is not None else q_codes.shape[0] // 2, want_rows)
    return m, sess


# ---- party mode: one party per process / GPU ---------------------

def _party_config(cfg: EngineConfig, own_prev, device: int) -> _Config:
    a, b = cfg.params()
    c = _Config()
    c.backend, c.variant, c.l, c.a, c.b, c.m = cfg.backend, cfg.variant, cfg.l, a, b, cfg.m
    c.rotations, c.debug_rows, c.match_ratio = cfg.rotations, 1 if cfg.debug_rows else 0, cfg.match_ratio
    op = np.ascontiguousarray(own_prev, np.uint8)
    for i in range(32):
        c.seeds[i] = int(op[i])
    c.device = device
    return c


def nccl_unique_id() -> bytes:
    out = np.zeros(128, np.uint8)
    if lib().irismpc_gpu_nccl_unique_id(out.ctypes.data_as(u8p)):
        raise DeviceError("NCCL is not available")
    return bytes(out)


class InProcNet:
    """InProcNet (transport.hpp:129-154): mailboxes for three parties in one process."""

    def __init__(self):
        h = vp()
        if lib().irismpc_gpu_inproc_create(C.byref(h)):
            raise DeviceError("inproc net")
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            lib().irismpc_gpu_inproc_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Party:
    """One MPC party (PartyCtx + Session<B,16,16>) on one GPU; its messages cross
    NCCL (nccl_id) or an InProcNet (net).  own_prev = seed_own (16 B) + seed_prev (16 B)."""

    def __init__(self, cfg: EngineConfig, party: int, own_prev, nccl_id: bytes | None = None,
                 net: InProcNet | None = None, device: int = 0):
        c = _party_config(cfg, own_prev, device)
        h = vp()
        if nccl_id is not None:
            idb = np.frombuffer(nccl_id, np.uint8).copy()
            rc = lib().irismpc_gpu_party_create_nccl(C.byref(c), party, idb.ctypes.data_as(u8p), C.byref(h))
        else:
            rc = lib().irismpc_gpu_party_create_inproc(C.byref(c), party, net._h, C.byref(h))
        if rc:
            raise _ERRORS.get(rc, IrisError)(f"party create failed ({rc})")
        self._h, self.cfg, self.party, self.s = h, cfg, party, 0
        self.rec = record_bytes(cfg.backend, cfg.l, cfg.variant)
        self.last_stats = PartyStats()
        self.row_bits = None

    def close(self):
        if getattr(self, "_h", None):
            lib().irismpc_gpu_party_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc):
        if rc:
            raise _ERRORS.get(rc, IrisError)(lib().irismpc_gpu_party_last_error(self._h).decode())

    def load_db(self, payload, s: int):
        a = np.ascontiguousarray(payload, np.uint8)
        self._check(lib().irismpc_gpu_party_load_db(self._h, a.ctypes.data, a.nbytes, s))
        self.s = s

    def batch_query(self, q, persons: int, want_rows: bool = False):
        a = np.ascontiguousarray(q, np.uint8)
        out = np.zeros(max(1, persons), np.uint8)
        rows = np.zeros(max(1, lane_count(persons, self.s, self.cfg.rotations)), np.uint8) if want_rows else None
        self._check(lib().irismpc_gpu_party_batch_query(self._h, a.ctypes.data, a.nbytes, persons, out.ctypes.data,
                                                        rows.ctypes.data if want_rows else None,
                                                        C.byref(self.last_stats)))
        self.row_bits = rows
        return out[:persons] if self.party == 1 else None

    def membership(self, q, want_rows: bool = False):
        a = np.ascontiguousarray(q, np.uint8)
        out = np.zeros(1, np.uint8)
        rows = np.zeros(max(1, self.s), np.uint8) if want_rows else None
        self._check(lib().irismpc_gpu_party_membership(self._h, a.ctypes.data, a.nbytes, out.ctypes.data,
                                                       rows.ctypes.data if want_rows else None,
                                                       C.byref(self.last_stats)))
        self.row_bits = rows
        return bool(out[0]) if self.party == 1 else None

    def read_tap(self, tap: int, n: int) -> np.ndarray:
        """DOT_*: this party's own additive dot [n] (plain-mask DOT_ML: the public
        popcount); others: [own, prev] x [n]."""
        kh, km, _ = VARIANT_WIDTHS[self.cfg.variant]
        if tap in (TAP_DOT_HD, TAP_DOT_ML):
            bits = kh if tap == TAP_DOT_HD else km
            out = np.zeros(n, np.uint32 if bits == 32 else np.uint16)
        elif tap == TAP_MSB:
            out = np.zeros(2 * n, np.uint8)
        else:
            out = np.zeros(2 * n, np.uint32)
        self._check(lib().irismpc_gpu_party_read_tap(self._h, tap, out.ctypes.data, out.nbytes))
        return out if tap in (TAP_DOT_HD, TAP_DOT_ML) else out.reshape(2, n)

    def stream_positions(self) -> np.ndarray:
        p = np.zeros(2, np.uint64)
        self._check(lib().irismpc_gpu_party_stream_positions(self._h, p.ctypes.data_as(u64p)))
        return p


def party_seeds(seeds48, party: int) -> np.ndarray:
    """(seed_own, seed_prev) of party 1..3 from seed_1 | seed_2 | seed_3 (rep3.hpp:124-127)."""
    s = np.ascontiguousarray(seeds48, np.uint8)
    p = party - 1
    q = (p + 2) % 3
    return np.concatenate([s[16 * p:16 * p + 16], s[16 * q:16 * q + 16]])


def run_parties_inproc(cfg: EngineConfig, seeds48, db_payloads, s: int, q_payloads, persons: int = 1,
                       membership: bool = False, want_rows: bool = False, device: int = 0):
    """run_parties (cluster.hpp:33-60) with one Party per host thread on one GPU,
    messages through an InProcNet.  Returns the three Party objects (P1 holds the result)."""
    import threading
    net = InProcNet()
    parties = [Party(cfg, p, party_seeds(seeds48, p), net=net, device=device) for p in (1, 2, 3)]
    results, errors = [None] * 3, [None] * 3

    def run(i):
        try:
            parties[i].load_db(db_payloads[i], s)
            if membership:
                results[i] = parties[i].membership(q_payloads[i], want_rows)
            else:
                results[i] = parties[i].batch_query(q_payloads[i], persons, want_rows)
        except Exception as e:  # noqa: BLE001 - surfaced below
            errors[i] = e

    th = [threading.Thread(target=run, args=(i,)) for i in range(3)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for e in errors:
        if e is not None:
            raise e
    parties[0].result = results[0]
    parties[0]._net = net  # keep the mailboxes alive with the parties
    return parties
