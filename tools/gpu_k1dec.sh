set -x
mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_k1w.py tests/test_gpu_forward.py -x -q > gpurun_out/pytest_k1dec.log 2>&1; rc=$?; echo rc=$rc
[ $rc -eq 0 ] || exit 1
timeout 300 python tools/bench_decode.py --specs 4:4 --batches 1,8,16 > gpurun_out/decode_k1.jsonl 2> gpurun_out/decode_k1.err; echo dec rc=$?
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --schedule serial > gpurun_out/bench_k1dec.log 2>&1; echo rc=$?
