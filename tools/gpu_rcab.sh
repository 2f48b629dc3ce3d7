# rank counts: histogram (default) vs radix-sort path, parity tests, then config 5
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_mocd.py tests/test_gpu_mocd_c5.py tests/test_gpu_calibrate.py -q -x 2>&1 | tail -2
SPLITQ_MOCD_RC_SORT=1 timeout 900 python -m pytest tests/test_gpu_mocd.py -q -x 2>&1 | tail -1
timeout 900 python tools/bench_c5.py > gpurun_out/c5_r02d.json 2> gpurun_out/c5_r02d.err; echo c5 rc=$?
