set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 900 python -m pytest tests/test_gpu_k1v3.py -x -q > gpurun_out/pytest_k1v3.log 2>&1; echo k1v3 rc=$?
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e > gpurun_out/bench.log 2>&1; echo bench rc=$?
