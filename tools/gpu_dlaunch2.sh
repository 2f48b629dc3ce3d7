# decode launch list at batch 1 / 16 (ncu flushes caches per kernel: weights come from HBM)
# with per-launch duration and DRAM bytes, plus the decode bench itself
mkdir -p gpurun_out
timeout 600 python tools/bench_decode.py --specs 4:4 --batches 1,16 > gpurun_out/dec_now.jsonl 2> gpurun_out/dec_now.err; echo dec rc=$?
for B in 1 16; do
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size,launch__block_size --clock-control none --csv --log-file gpurun_out/dl2_b$B.csv \
  python tools/bench_decode.py --specs 4:4 --batches $B --iters 1 > gpurun_out/dl2_b$B.log 2>&1; echo ncu rc=$?
done
