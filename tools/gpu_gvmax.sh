set -x
mkdir -p gpurun_out
SPLITQ_GEMV_MAX_ROWS=32 timeout 300 python tools/bench_decode.py --specs 4:4 --batches 8,16,32 > gpurun_out/decode_gv32.jsonl 2> gpurun_out/decode_gv32.err; echo dec rc=$?
