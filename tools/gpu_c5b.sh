# config 5 after the text-score compaction + the MOCD / calibration GPU tests
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_mocd.py tests/test_gpu_mocd_c5.py tests/test_gpu_calibrate.py -q -x 2>&1 | tail -2
timeout 900 python tools/bench_c5.py > gpurun_out/c5_r02e.json 2> gpurun_out/c5_r02c.err; echo c5 rc=$?
