# K1 phase clocks at decode sizes: a -DKW_TRACE build, then the trace tool
set -x
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_k1w.py -x -q > gpurun_out/pytest_k1w.log 2>&1; echo k1w rc=$?
SPLITQ_NVCC_EXTRA=-DKW_TRACE python -c "import __graft_entry__ as g; g.build()" > gpurun_out/k1trace_build.log 2>&1; echo build rc=$?
SPLITQ_K1_WPR=8 timeout 300 python tools/k1_trace.py q gate down > gpurun_out/k1trace.log 2>&1; echo trace rc=$?
SPLITQ_K1_WPR=16 timeout 300 python tools/k1_trace.py q gate down > gpurun_out/k1trace16.log 2>&1; echo trace rc=$?
