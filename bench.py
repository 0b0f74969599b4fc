#!/usr/bin/env python3
"""Benchmark: iris comparisons/sec of the full 3-party mpc-lift query on B200.

A step is one complete batch query of BASELINE.json configs[1]: 32 query eye
codes (16 persons) x 31 rotations against a 100k-row synthetic DB per GPU,
12800-bit codes + masks, all three parties' shares resident in HBM:
query-share broadcast -> K1 prep -> K2 tcgen05 limb GEMMs -> K4 threshold
(reshare, lift, MSB) -> K5 MPC-OR -> open of one bit per person at P1.
comparisons = codes * 31 * DB rows (inner-batch pair lanes are computed but
not counted).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (DB sharded, weak scaling)
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

L = 12800
ROT = 31
PERSONS = 16            # 32 eye codes
ROWS_PER_GPU = 100_000  # configs[1]
METRIC = "iris comparisons/sec (query x rotation x DB)"
UNIT = "comparisons/s"
VARIANTS = {"plain-mask": 0, "mpc-lift": 1, "const-lift": 2, "no-lift": 3}
LIMB_PRODUCTS = {0: 0, 16: 3, 32: 10}  # u8-limb MMAs per k-step of a Z_2^K dot (gemm.cu)
WIDTHS = {0: (16, 0), 1: (16, 16), 2: (16, 32), 3: (32, 32)}


def ops_per_lane(backend: int, variant: int = 1) -> int:
    """int8 tensor ops per comparison lane, all 3 parties (460,800
    for mpc-lift Shamir, 921,600 replicated); the public-mask popcount is one
    party-independent 1-limb GEMM with K = l."""
    kh, km = WIDTHS[variant]
    k = L if backend == 1 else 2 * L
    macs = 3 * LIMB_PRODUCTS[kh] * k + (3 * LIMB_PRODUCTS[km] * k if km else L)
    return 2 * macs
ALG_BYTES_PER_LANE = 12.75               # compare/reduce phase


def prf_blocks_per_lane(variant: int = 1) -> float:
    """ChaCha12 blocks per comparison lane of the reference-exact PRF layout
    (DESIGN §4): reshare 1 u64 per seed per shared dot, bit_inject
    4 u64 per inject (mpc-lift only), one u64 per seed per 64-lane word per AND
    gate (lift 64 + msb 61 for mpc-lift; msb only otherwise)."""
    reshare = 3 * (1 if variant == 0 else 2) / 8
    inject = 1.0 if variant == 1 else 0.0
    gates = {0: 29, 1: 125, 2: 61, 3: 61}[variant]
    return reshare + inject + gates * 3 / 512


def env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


class Clocks:
    """One `nvidia-smi -lms 200` sampler (clocks + throttle reasons) running
    during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,power.draw")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.samples = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is None:
            return
        time.sleep(0.25)
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        for line in out.splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 7:
                self.samples.append(parts)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i].lower() == "active"})
        pw = []
        for s in self.samples:
            try:
                pw.append(float(s[6]))
            except ValueError:
                pass
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples),
                "power_w_median": statistics.median(pw) if pw else None, "power_w_max": max(pw) if pw else None}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


def chacha_peak():
    """measured ChaCha12 keystream rate of this device (tools/chacha_peak.cu)"""
    p = os.path.join(ROOT, "profiles", "chacha_peak.json")
    if os.path.exists(p):
        try:
            return json.load(open(p))["chacha12_blocks_per_s_store"]
        except Exception:
            return None
    return None


def ncu_traffic(rp: bool = False):
    """dram bytes per GEMM launch from the committed ncu --set full capture (or None);
    rp: the rotation-pair GEMM launches"""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(p):
        try:
            d = json.load(open(p))
            if rp and "rotation_pair" in d:
                d = d["rotation_pair"]
            return d.get("gemm_dram_bytes_per_launch"), d.get("tensor_pipe_active_pct")
        except Exception:
            return None, None
    return None, None


# ------------------------------------------------------------------ CPU baseline

def cpu_reference_rate(backend: int, rows: int, persons: int, steps: int, variant: int = 1):
    """The reference (oracle/_ref, compiled from the reference sources) on the
    host cores: run_parties + party_batch_query per step; QueryStats.wall_ms."""
    from oracle import pyoracle as O
    import ctypes as C
    cores = os.cpu_count() or 1
    if O.ref_available():
        # all host threads: torchrun exports OMP_NUM_THREADS=1 to every rank, and the
        # reference's OpenMP dot loop (libgomp) would otherwise run on one core
        os.environ["OMP_NUM_THREADS"] = str(cores)
        R = O.ref()
        try:
            C.CDLL("libgomp.so.1").omp_set_num_threads(C.c_int(cores))
        except OSError:
            pass
        h = R.ref_bench_prepare(backend, variant, L, rows, persons)
        times = []
        m0 = C.c_uint8(0)
        for _ in range(steps):
            times.append(R.ref_bench_step(h, C.byref(m0)))
        R.ref_bench_free(h)
        ms = statistics.median(times)
        cmp_ = 2 * persons * ROT * rows
        return {"value": cmp_ / (ms / 1e3), "unit": UNIT, "cores": cores, "kind": "reference",
                "sample": f"reference run_batch (oracle/_ref, OpenMP parallel_dot, all {cores} host threads): "
                          f"{2 * persons} codes x {ROT} rot x {rows} rows, median of {steps} steps of "
                          f"QueryStats.wall_ms={ms:.0f} ms; linear in rows",
                "planted_match": int(m0.value)}
    # port: the C restatement, single thread
    rng = O.Rng(2)
    dc, dm = O.records(rng, L, rows, 0.9)
    qc, qm = O.records(rng, L, 2 * persons, 0.9)
    cfg = O.make_config(backend, L, variant=variant)
    t0 = time.perf_counter()
    O.run_local(cfg, 7, dc, dm, qc, qm, persons)
    dt = time.perf_counter() - t0
    return {"value": 2 * persons * ROT * rows / dt, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"oracle C port incl. dealing: {2 * persons} codes x {ROT} rot x {rows} rows"}


def run_reference_arm(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    backend = 1 if args.backend == "shamir" else 0
    rows = args.ref_rows
    for _ in range(args.warmup and 1):
        pass
    variant = VARIANTS[args.variant]
    res = cpu_reference_rate(backend, rows, 1, max(1, args.steps), variant)
    line = {"metric": METRIC, "value": res["value"], "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 2 * ROT * rows / res["value"] * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u16", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": f"cfg2-shape sample: 1 person (2 codes) x {ROT} rot x {rows} rows, "
                                   f"l={L}, {args.variant}, {args.backend}", "l": L, "rotations": ROT,
                       "variant": args.variant},
            "cpu_baseline": {k: res[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": res["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def compare_roofline(span_ms: float, lanes: int, variant: int, peaks: dict) -> dict:
    """The compare/reduce phase (reshare -> lift -> MSB -> OR) against both of
    its ceilings over the threshold stream's span: HBM at the SURVEY §8d
    algorithmic 12.75 B/lane, and the ALU pipe as ChaCha12 blocks/s against the
    measured keystream rate (profiles/chacha_peak.json).  The PRF layout is the
    reference's (2.48 blocks/lane for mpc-lift), so the phase is ALU-bound."""
    sec = max(span_ms, 1e-9) / 1e3
    hbm = ALG_BYTES_PER_LANE * lanes / sec / 1e9
    blocks = prf_blocks_per_lane(variant) * lanes
    cp = chacha_peak()
    out = {"bound": "alu", "kernels": "k_gate_keystream, k_reshare, k_lift, k_inject, k_msb",
           "hbm": {"achieved": hbm, "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": hbm / peaks["hbm_gbs"],
                   "alg_bytes_per_lane": ALG_BYTES_PER_LANE},
           "chacha": {"achieved": blocks / sec, "peak": cp, "unit": "ChaCha12 blocks/s",
                      "frac": (blocks / sec / cp) if cp else None,
                      "blocks_per_lane": prf_blocks_per_lane(variant)},
           "span_ms": span_ms,
           "note": "over the threshold stream span, which overlaps the GEMM; the GEMM and the "
                   "ChaCha work share the 1000 W power cap and do not overlap in time on the "
                   "same SMs (DESIGN.md section 4), so the span is mostly GEMM-bound time"}
    return out


# ------------------------------------------------------------------ GPU arm

def main_gpu(args):
    import torch
    import torch.distributed as dist
    import paper_2405_04463_b200 as P
    from paper_2405_04463_b200.dist import shard_rows, sharded_batch_query

    rank, world, local = env_rank()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    backend = P.SHAMIR if args.backend == "shamir" else P.REPLICATED
    S = args.rows * world
    row_off, rows = shard_rows(S, world, rank)
    persons = args.persons
    ncodes = 2 * persons
    variant = VARIANTS[args.variant]
    cfg = P.EngineConfig(backend=backend, l=L, rotations=ROT, variant=variant)
    sess = P.Session(cfg, master_seed=7, device=local, shard_rank=rank, db_rows_total=S if world > 1 else 0,
                     db_row_offset=row_off)
    t0 = time.time()
    sess.synth_db(rows, rng_seed=2, first=row_off, mask_density=0.9, deal_seed=7)
    setup_s = time.time() - t0

    # query records: Rng(2) records after the DB; person 0's left eye = DB row S/2
    # rotated by +2 strides with 4 flipped code bits (planted near-match)
    wl = L // 64
    qpay = [torch.empty(ncodes * sess.rec, dtype=torch.uint8, device="cuda") for _ in range(3)]
    if rank == 0:
        codes = torch.empty((ncodes, wl), dtype=torch.int64, device="cuda")
        masks = torch.empty((ncodes, wl), dtype=torch.int64, device="cuda")
        sess.synth_records(2, S, ncodes, 0.9, codes, masks)
        # the planted row may live on another shard: regenerate it from the stream
        rc_ = torch.empty((1, wl), dtype=torch.int64, device="cuda")
        rm_ = torch.empty((1, wl), dtype=torch.int64, device="cuda")
        sess.synth_records(2, S // 2, 1, 0.9, rc_, rm_)
        c = np.unpackbits(rc_.cpu().numpy().view(np.uint8), bitorder="little")
        m = np.unpackbits(rm_.cpu().numpy().view(np.uint8), bitorder="little")
        by = 2 * (L // 64)
        c, m = np.roll(c, by), np.roll(m, by)
        for f in range(4):
            c[f * (L // 4) + 7] ^= 1
        codes[0] = torch.from_numpy(np.packbits(c, bitorder="little").view(np.int64).copy())
        masks[0] = torch.from_numpy(np.packbits(m, bitorder="little").view(np.int64).copy())
        sess.deal_payload(7, 2, 0, codes, masks, qpay)
    host_q = [torch.empty(ncodes * sess.rec, dtype=torch.uint8).pin_memory() for _ in range(3)]
    if rank == 0:
        for h, d in zip(host_q, qpay):
            h.copy_(d.cpu())
    parts = torch.zeros((world, 3, persons), dtype=torch.uint8, device="cuda")
    ext = torch.cuda.ExternalStream(sess.stream)

    def step(from_host: bool):
        if world == 1:
            if from_host:
                return sess.batch_query([h.numpy() for h in host_q], persons)
            return sess.batch_query(qpay, persons)
        if from_host and rank == 0:
            for d, h in zip(qpay, host_q):
                d.copy_(h, non_blocking=True)
        return sharded_batch_query(sess, qpay, persons, dist, world, rank, parts)

    for _ in range(args.warmup):
        out = step(False)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()

    stats_acc = {"gemm_ms": 0.0, "launches": 0, "gemm_launches": 0, "gemm_ops": 0, "rp": 0}
    with Clocks(local) as clk:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(ext):
            ev0.record()
        h0 = time.perf_counter()
        for _ in range(args.steps):
            out = step(False)
            st = sess.last_stats
            stats_acc["gemm_ms"] += st.gemm_ms
            stats_acc["launches"] += st.kernel_launches + (1 if world > 1 and rank == 0 else 0)
            stats_acc["gemm_launches"] += st.gemm_launches
            stats_acc["gemm_ops"] += st.gemm_int8_ops
            stats_acc["rp"] = int(st.rotation_pair_gemm)
        with torch.cuda.stream(ext):
            ev1.record()
        torch.cuda.synchronize()
        host_s = time.perf_counter() - h0
        if world > 1:
            dist.barrier()
    dev_ms = ev0.elapsed_time(ev1) / args.steps
    t = torch.tensor([dev_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    planted = int(out[0]) if out is not None else None

    # e2e through the public API from pinned host buffers (H2D + D2H inside)
    e2e_ms = []
    for _ in range(max(2, args.steps // 2)):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        a = time.perf_counter()
        step(True)
        torch.cuda.synchronize()
        e2e_ms.append((time.perf_counter() - a) * 1e3)
    e2e = torch.tensor([statistics.median(e2e_ms)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(e2e, op=dist.ReduceOp.MAX)

    lanes_db = ncodes * ROT * S
    value = lanes_db / (ms / 1e3)
    if rank == 0:
        peaks, src = load_peaks()
        gemm_ms = stats_acc["gemm_ms"] / max(1, stats_acc["gemm_launches"])
        local_lanes = ncodes * ROT * rows
        opl = ops_per_lane(backend, variant)
        kh, km = WIDTHS[variant]
        plane_kb = L * (3 * kh // 8 + (3 * km // 8 if km else 1)) / 1e3
        ops_launch = local_lanes * opl / max(1, stats_acc["gemm_launches"] // args.steps)
        achieved = ops_launch / (gemm_ms / 1e3) / 1e12
        exec_opl = stats_acc["gemm_ops"] / max(1, args.steps) / max(1, local_lanes)
        exec_tops = stats_acc["gemm_ops"] / max(1, stats_acc["gemm_launches"]) / (gemm_ms / 1e3) / 1e12
        i8 = os.path.join(ROOT, "profiles", "int8_peak.json")
        if os.path.exists(i8):
            peak = json.load(open(i8))["int8_tops_burst"]
            peak_note = "measured cuBLASLt int8 burst (profiles/int8_peak.json, tools/measure_int8_peak.py)"
        else:
            peak = 2.0 * peaks["bf16_tflops"]
            peak_note = f"2 x {src} bf16 ({peaks['bf16_tflops']} TF/s); dense int8 = 2x bf16 on sm_100"
        cpu = cpu_reference_rate(backend, args.ref_rows, 1, 1, variant) if (world == 1 and not args.no_cpu) else None
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": f"configs[1]: {ncodes} query codes ({persons} persons) x {ROT} rotations vs "
                                   f"{rows} DB rows per GPU (total {S}), l={L}, 3-party {args.variant}, "
                                   f"{args.backend} backend", "l": L, "rotations": ROT, "persons": persons,
                       "db_rows_total": S, "db_rows_per_gpu": rows, "backend": args.backend,
                       "variant": args.variant,
                       "l2": f"inputs larger than L2 (DB limb planes {plane_kb:.1f} KB/row resident in HBM)",
                       "parallelism": f"db-shard x{world}"},
            "e2e": {"value": lanes_db / (float(e2e.item()) / 1e3), "unit": UNIT,
                    "h2d_bytes_per_step": 3 * ncodes * sess.rec, "d2h_bytes_per_step": persons,
                    "note": "median of single queries through the public API (pinned host payloads in, "
                            "person_match out), each bracketed by a host sync; the GPU idles between "
                            "them, so under the 1000 W cap a single query can run at higher clocks "
                            "than the back-to-back steps behind `value`"},
            "roofline": {"bound": "tensor", "kernel": "k_limb_gemm_pair (tcgen05.mma.cta_group::2.kind::i8)",
                         "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                         "traffic": ncu_traffic(bool(stats_acc["rp"]))[0],
                         "ncu_tensor_pipe_active_pct": ncu_traffic(bool(stats_acc["rp"]))[1],
                         "executed": {"int8_ops_per_lane": exec_opl, "achieved": exec_tops, "frac": exec_tops / peak,
                                      "rotation_pair_gemm": bool(stats_acc["rp"])},
                         "note": f"achieved = algorithmic int8 ops ({opl}/lane) / GEMM time; peak = {peak_note}. "
                                 "The rotation-pair (Winograd F(2,2)) GEMMs execute fewer int8 MACs than the "
                                 "algorithmic count (DESIGN.md section 8), so `achieved` can exceed the executed "
                                 "rate: `executed` is the tensor-pipe figure"},
            "gpu_launches": stats_acc["launches"],
            "clocks": clk.summary(),
            "roofline_compare": compare_roofline(sess.last_stats.threshold_ms, local_lanes, variant, peaks),
            "phase_ms": {"gemm_per_launch": gemm_ms,
                         "gemm_launches_per_step": stats_acc["gemm_launches"] / args.steps,
                         "threshold_stream_span": sess.last_stats.threshold_ms,
                         "or": sess.last_stats.or_ms, "prep": sess.last_stats.prep_ms, "step": ms,
                         "host_wall_per_step": host_s / args.steps * 1e3,
                         "note": "GEMM (stream 1) and threshold (stream 2) overlap; the span is the "
                                 "threshold stream's first-start to last-end time of the last step"},
            "planted_match": planted, "setup_s": setup_s,
        }
        if cpu is not None:
            line["cpu_baseline"] = {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample")}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--backend", default="shamir", choices=["shamir", "replicated"])
    ap.add_argument("--variant", default="mpc-lift", choices=list(VARIANTS))
    ap.add_argument("--rows", type=int, default=ROWS_PER_GPU)
    ap.add_argument("--persons", type=int, default=PERSONS)
    ap.add_argument("--ref-rows", type=int, default=3000, dest="ref_rows")
    ap.add_argument("--no-cpu", action="store_true", dest="no_cpu")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference_arm(args)
    return main_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
