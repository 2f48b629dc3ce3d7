set -x
mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_k1w.py tests/test_gpu_forward.py -x -q > gpurun_out/pytest_g64.log 2>&1; rc=$?; echo rc=$rc
[ $rc -eq 0 ] || exit 1
B="python bench.py --no-e2e --no-cpu-baseline --steps 5 --warmup 3"
timeout 600 $B > gpurun_out/bench_g64_a4.log 2>&1
timeout 600 $B --abits 8 > gpurun_out/bench_g64_a8.log 2>&1; echo rc=$?
