set -x
mkdir -p gpurun_out
SPLITQ_GEMV_MAX_ROWS=32 timeout 300 python tools/bench_decode.py --specs 4:4 --batches 24,32 > gpurun_out/decode_gv32.jsonl 2> gpurun_out/decode_gv32.err; echo dec rc=$?
timeout 300 python tools/bench_decode.py --specs 4:4 --batches 24,32 > gpurun_out/decode_tc32.jsonl 2> gpurun_out/decode_tc32.err; echo dec rc=$?
