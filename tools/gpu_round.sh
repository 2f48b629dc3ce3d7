# round check: all GPU tests, bench (prefill), decode bench
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; rc=$?; echo pytest rc=$rc
[ $rc -eq 0 ] || exit 1
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; echo bench rc=$?
timeout 300 python tools/bench_decode.py --specs 4:4 > gpurun_out/decode_gv.jsonl 2> gpurun_out/decode_gv.err; echo dec rc=$?
