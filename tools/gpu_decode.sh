# decode-path check: GPU parity of the forward / K1 tests, stage micro-timings
# and the config-4 decode bench (stops after a failing test run)
set -x
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_forward.py tests/test_gpu_k1w.py -x -q > gpurun_out/pytest_fwd.log 2>&1; rc=$?
echo fwd rc=$rc
[ $rc -eq 0 ] || exit 1
timeout 200 python tools/decode_micro.py --batches 1,2,4,8,16,64 > gpurun_out/dmicro_gv.log 2>&1; echo micro rc=$?
timeout 300 python tools/bench_decode.py --specs 4:4 > gpurun_out/decode_gv.jsonl 2> gpurun_out/decode_gv.err; echo dec rc=$?
