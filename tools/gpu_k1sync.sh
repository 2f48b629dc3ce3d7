set -x
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_k1w.py -x -q > gpurun_out/pytest_k1s.log 2>&1; echo rc=$?
for V in "128 0" "128 1" "256 1" "512 1" "256 0"; do
  set -- $V
  SPLITQ_NVCC_EXTRA="-DKW_THREADS_N=$1 -DKW_SYNC_ROWS=$2" python -c "import __graft_entry__ as g; g.build()" > gpurun_out/k1s_build.log 2>&1
  timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --schedule serial > gpurun_out/bench_k1s_$1_$2.log 2>&1; echo rc=$?
done
