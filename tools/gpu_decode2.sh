set -x
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_forward.py tests/test_gpu_layer_io.py -x -q > gpurun_out/pytest_fwd.log 2>&1; rc=$?; echo fwd rc=$rc
[ $rc -eq 0 ] || exit 1
timeout 300 python tools/bench_decode.py --specs 4:4 > gpurun_out/decode_gv.jsonl 2> gpurun_out/decode_gv.err; echo dec rc=$?
