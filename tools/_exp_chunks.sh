b() { n=$1; shift; timeout 600 python bench.py "$@" --no-cpu > gpurun_out/$n.log 2>&1; echo rc=$? >> gpurun_out/$n.log; }
b f16 --rows 1000000 --persons 8 --steps 5 --warmup 3
b f64 --rows 1000000 --persons 32 --steps 5 --warmup 3
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests3.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests3.log
timeout 400 python bench.py > gpurun_out/bench_final.log 2>&1; echo rc=$? >> gpurun_out/bench_final.log
