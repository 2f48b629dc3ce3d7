# calibration caller parity, then the sanitizer pass on the small kernel cases
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_calibrate.py tests/test_build_layer_golden.py -q > gpurun_out/pytest_cal.log 2>&1; echo pytest rc=$?
tail -15 gpurun_out/pytest_cal.log
timeout 300 python tools/sanitize.py > gpurun_out/san_plain.log 2>&1; echo plain rc=$?; tail -2 gpurun_out/san_plain.log
timeout 1200 compute-sanitizer --tool memcheck --leak-check full --error-exitcode 9 python tools/sanitize.py > gpurun_out/san_memcheck.log 2>&1; echo memcheck rc=$?
tail -6 gpurun_out/san_memcheck.log
