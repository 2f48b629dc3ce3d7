set -x
timeout 900 python -m pytest tests/test_gpu_k1w.py tests/test_gpu_forward.py -q > gpurun_out/pytest_k1w.log 2>&1; echo tests rc=$?
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo bench rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:splitq_gemm2 -s 0 -c 2 -o gpurun_out/lr1_full python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_lr1.log 2>&1; echo ncu rc=$?
