set -x
mkdir -p gpurun_out
SPLITQ_NVCC_EXTRA=-DG2_TRACE python -c "import __graft_entry__ as g; g.build()" > gpurun_out/g2t_build.log 2>&1; echo build rc=$?
SPLITQ_TRACE_MODE=2 timeout 300 python tools/lr1_trace.py q gate > gpurun_out/lr1trace.log 2>&1
SPLITQ_TRACE_MODE=0 timeout 300 python tools/lr1_trace.py q >> gpurun_out/lr1trace.log 2>&1; echo rc=$?
