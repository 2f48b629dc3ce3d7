set -x
mkdir -p gpurun_out
for GM in 32 64 128; do
SPLITQ_TILE_GM=$GM timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --schedule serial > gpurun_out/bench_gm$GM.log 2>&1; echo rc=$?
done
