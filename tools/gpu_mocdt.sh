set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_mocd.py -x -q > gpurun_out/pytest_mocd.log 2>&1; echo rc=$?
