set -x
mkdir -p gpurun_out
s0=$(date +%s); timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q > gpurun_out/pytest_full.log 2>&1; echo rc=$? secs=$(( $(date +%s) - s0 ))
