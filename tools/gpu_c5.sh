set -x
mkdir -p gpurun_out
timeout 1500 python tools/bench_c5.py > gpurun_out/c5.json 2> gpurun_out/c5.err; echo rc=$?
