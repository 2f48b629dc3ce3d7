set -x
mkdir -p gpurun_out
for i in 1 2; do
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --schedule serial > gpurun_out/bench_serial_$i.log 2>&1; echo rc=$?
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --schedule branches > gpurun_out/bench_branches_$i.log 2>&1; echo rc=$?
done
