set -x
mkdir -p gpurun_out
s0=$(date +%s); timeout 900 python bench.py > gpurun_out/bench_default.log 2> gpurun_out/bench_default.err; echo bench rc=$? secs=$(( $(date +%s) - s0 ))
