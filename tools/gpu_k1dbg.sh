set -x
mkdir -p gpurun_out
SPLITQ_NVCC_EXTRA=-DKW_DEBUG python -c "import __graft_entry__ as g; g.build()" > gpurun_out/k1dbg_build.log 2>&1
timeout 300 python tools/k1_debug.py 4 > gpurun_out/k1dbg.log 2>&1
timeout 300 python tools/k1_debug.py 8 >> gpurun_out/k1dbg.log 2>&1; echo rc=$?
