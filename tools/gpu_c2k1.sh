set -x
mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_forward.py -x -q > gpurun_out/pytest_fwd.log 2>&1; echo rc=$?
B="python bench.py --no-e2e --no-cpu-baseline --model 3b --tokens 4096 --steps 20 --warmup 5"
timeout 600 $B > gpurun_out/c2k1_def.log 2>&1; echo rc=$?
timeout 600 python bench.py --no-e2e --no-cpu-baseline --tokens 4096 --steps 10 --warmup 3 --schedule serial > gpurun_out/c3_4096.log 2>&1; echo rc=$?
