set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_mocd.py -x -q > gpurun_out/pytest_mocd.log 2>&1; rc=$?; echo rc=$rc
[ $rc -eq 0 ] || exit 1
timeout 1500 python tools/bench_c5.py > gpurun_out/c5.json 2> gpurun_out/c5.err; echo rc=$?
