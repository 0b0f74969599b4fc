#!/usr/bin/env python3
"""Time and energy per configs[1] query (NVML total-energy counter), optionally
next to a pure-ALU ChaCha12 load on a second stream (co-running
analysis).

    python tools/energy_query.py                      # full query: ms, J, W
    python tools/energy_query.py --corun 246000000    # + 2.46e8 ChaCha12 blocks per query
    python tools/energy_query.py --chacha-only 246000000 --grid 148

The library under test is whatever paper_2405_04463_b200/libirismpc_gpu.so is
(the A/B builds of DESIGN.md §4 compile single kernels out of that library).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
BUILD = os.path.join(ROOT, "tools", "_build")
LOAD_SO = os.path.join(BUILD, "libchacha_launch.so")


def load_lib():
    src = os.path.join(ROOT, "tools", "chacha_launch.cu")
    if not os.path.exists(LOAD_SO) or os.path.getmtime(LOAD_SO) < os.path.getmtime(src):
        os.makedirs(BUILD, exist_ok=True)
        subprocess.run(["nvcc", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-Xcompiler", "-fPIC",
                        "-shared", "-I", os.path.join(ROOT, "paper_2405_04463_b200", "csrc"), src, "-o", LOAD_SO],
                       check=True)
    L = C.CDLL(LOAD_SO)
    L.chacha_load.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint, C.c_uint, C.c_void_p]
    return L


class ClockSampler:
    """SM clock every 2 ms during a measurement (NVML)."""

    def __init__(self, nvml, h):
        self.nvml, self.h, self.s, self.on = nvml, h, [], False

    def __enter__(self):
        self.on = True

        def f():
            while self.on:
                self.s.append(self.nvml.nvmlDeviceGetClockInfo(self.h, self.nvml.NVML_CLOCK_SM))
                time.sleep(0.002)

        self.t = threading.Thread(target=f)
        self.t.start()
        return self

    def __exit__(self, *a):
        self.on = False
        self.t.join()

    def median(self):
        return sorted(self.s)[len(self.s) // 2] if self.s else None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--queries", type=int, default=200)
    ap.add_argument("--rows", type=int, default=100_000)
    ap.add_argument("--persons", type=int, default=16)
    ap.add_argument("--corun", type=int, default=0, help="ChaCha12 blocks launched next to each query")
    ap.add_argument("--chacha-only", type=int, default=0, dest="chacha_only")
    ap.add_argument("--grid", type=int, default=0, help="ChaCha load grid (0: one thread per block)")
    ap.add_argument("--threads", type=int, default=256)
    a = ap.parse_args()

    import pynvml
    import torch
    import paper_2405_04463_b200 as P

    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    sink = torch.zeros(4, dtype=torch.uint8, device="cuda")
    s2 = torch.cuda.Stream()
    load = load_lib() if (a.corun or a.chacha_only) else None

    def chacha(n, i):
        load.chacha_load(C.c_void_p(s2.cuda_stream), n, i * n, a.grid, a.threads, C.c_void_p(sink.data_ptr()))

    if a.chacha_only:
        fn = lambda i: chacha(a.chacha_only, i)  # noqa: E731
    else:
        L = 12800
        sess = P.Session(P.EngineConfig(backend=P.SHAMIR, l=L, rotations=31), master_seed=7, device=0)
        sess.synth_db(a.rows, rng_seed=2, first=0, mask_density=0.9, deal_seed=7)
        n = 2 * a.persons
        q = [torch.empty(n * sess.rec, dtype=torch.uint8, device="cuda") for _ in range(3)]
        codes = torch.empty((n, L // 64), dtype=torch.int64, device="cuda")
        masks = torch.empty_like(codes)
        sess.synth_records(2, a.rows, n, 0.9, codes, masks)
        sess.deal_payload(7, 2, 0, codes, masks, q)

        def fn(i):
            if a.corun:
                chacha(a.corun, i)
            sess.batch_query(q, a.persons)

    for i in range(3):
        fn(i)
    torch.cuda.synchronize()
    time.sleep(1.0)
    clk = ClockSampler(pynvml, h)
    with clk:
        e0 = pynvml.nvmlDeviceGetTotalEnergyConsumption(h)
        t0 = time.perf_counter()
        for i in range(a.queries):
            fn(i)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        e1 = pynvml.nvmlDeviceGetTotalEnergyConsumption(h)
    dt = t1 - t0
    print(json.dumps({"ms_per_query": dt / a.queries * 1e3, "J_per_query": (e1 - e0) / 1e3 / a.queries,
                      "avg_W": (e1 - e0) / 1e3 / dt, "sm_mhz_median": clk.median(), "queries": a.queries,
                      "corun_blocks": a.corun, "chacha_only_blocks": a.chacha_only, "grid": a.grid,
                      "threads": a.threads}))


if __name__ == "__main__":
    main()
