SPLITQ_NVCC_EXTRA=-DKW_DEBUG python paper_2605_19929_b200/_build.py --force > gpurun_out/dbg_build.log 2>&1
python tools/k1_debug.py > gpurun_out/k1_debug.log 2>&1; echo rc=$?
