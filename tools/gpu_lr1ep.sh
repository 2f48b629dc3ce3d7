set -x
mkdir -p gpurun_out
timeout 500 python -m pytest tests/test_gpu_forward.py tests/test_gpu_fullsize.py tests/test_gpu_gemm.py -x -q > gpurun_out/pytest_lr1ep.log 2>&1; rc=$?; echo rc=$rc
[ $rc -eq 0 ] || exit 1
timeout 600 python bench.py --no-e2e --no-cpu-baseline --steps 5 --warmup 3 --schedule serial > gpurun_out/bench_lr1ep.log 2>&1; echo rc=$?
SPLITQ_NVCC_EXTRA=-DG2_TRACE python -c "import __graft_entry__ as g; g.build()" > gpurun_out/g2t_build.log 2>&1
SPLITQ_TRACE_MODE=2 timeout 300 python tools/lr1_trace.py q > gpurun_out/lr1trace.log 2>&1; echo rc=$?
