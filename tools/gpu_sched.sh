set -x
mkdir -p gpurun_out
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --schedule serial > gpurun_out/bench_serial.log 2>&1; echo rc=$?
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --schedule branches > gpurun_out/bench_branches.log 2>&1; echo rc=$?
