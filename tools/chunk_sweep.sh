#!/usr/bin/env bash
# Row-chunk size sweep behind profiles/r1_scaling.md ("Plain-GEMM row chunks on large DBs").
# Run on one B200 from the repo root, e.g.
#   gpurun --timeout 1200 -- 'bash tools/chunk_sweep.sh'
# Each line: bench.py at 1M DB rows with the default chunk rule, then with IRISMPC_CHUNK_LANES forced.
set -u
mkdir -p gpurun_out
b() { n=$1; shift; timeout 600 python bench.py "$@" --no-cpu > gpurun_out/$n.log 2>&1; echo rc=$? >> gpurun_out/$n.log; }
for persons in 4 8 16 32; do
  b sweep_p${persons}_default --rows 1000000 --persons $persons --steps 5 --warmup 3
  for L in 16777216 33554432 67108864 134217728; do
    IRISMPC_CHUNK_LANES=$L b sweep_p${persons}_$L --rows 1000000 --persons $persons --steps 5 --warmup 3
  done
done
