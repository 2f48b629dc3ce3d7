set -x
mkdir -p gpurun_out
SPLITQ_NVCC_EXTRA=-DTS_TRACE python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ts_build.log 2>&1
timeout 900 python tools/bench_c5.py > gpurun_out/c5_trace.json 2> gpurun_out/c5_trace.err; echo rc=$?
grep TS_TRACE gpurun_out/c5_trace.json gpurun_out/c5_trace.err | head -20
