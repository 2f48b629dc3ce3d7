set -x
mkdir -p gpurun_out
timeout 600 python tools/ts_repro.py 196608 18755 3 > gpurun_out/ts1.log 2>&1; echo rc=$?
timeout 600 python tools/ts_repro.py 196608 64 3 check > gpurun_out/ts2.log 2>&1; echo rc=$?
timeout 900 compute-sanitizer --tool memcheck --print-limit 5 python tools/ts_repro.py 196608 300 3 > gpurun_out/ts3.log 2>&1; echo rc=$?
