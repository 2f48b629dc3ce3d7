# K1 decode phase clocks (KW_TRACE build on the box; the box copy is discarded)
mkdir -p gpurun_out
SPLITQ_NVCC_EXTRA=-DKW_TRACE python -c "from paper_2605_19929_b200 import _build; _build.build(force=True)" > gpurun_out/k1trace_build.log 2>&1; echo build rc=$?
SPLITQ_K1_WPR=8 timeout 300 python tools/k1_trace.py q down > gpurun_out/k1trace.log 2>&1; echo trace rc=$?
cat gpurun_out/k1trace.log | grep -v Warn
