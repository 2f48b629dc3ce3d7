# decode launch list (warm caches): kernel durations of graph-replayed decode steps
set -x
mkdir -p gpurun_out
for B in ${BATCHES:-1 8}; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/dlaunch_b$B.csv \
  python tools/bench_decode.py --specs 4:4 --batches $B --iters 2 > gpurun_out/dlaunch_b$B.log 2>&1; echo ncu rc=$?
done
