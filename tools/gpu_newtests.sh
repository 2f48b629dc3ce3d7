mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_ops.py tests/test_gpu_mocd_c5.py tests/test_build_layer_golden.py tests/test_gpu_forward.py tests/test_gpu_fullsize.py -q -x > gpurun_out/pytest_new.log 2>&1; echo rc=$?
tail -25 gpurun_out/pytest_new.log
