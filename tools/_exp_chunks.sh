b() { n=$1; shift; timeout 600 python bench.py "$@" --no-cpu > gpurun_out/$n.log 2>&1; echo rc=$? >> gpurun_out/$n.log; }
b d2_new --rows 1000000 --persons 32 --steps 5 --warmup 3
IRISMPC_CHUNK_LANES=134217728 b d2_27 --rows 1000000 --persons 32 --steps 5 --warmup 3
b d2_256 --rows 1000000 --persons 128 --steps 3 --warmup 3
IRISMPC_RP=0 b d1_plain --steps 20 --warmup 3
b d1 --steps 20 --warmup 3
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests2.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests2.log
