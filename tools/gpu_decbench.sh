# bench.py --decode lines (config 4 decode regime)
mkdir -p gpurun_out
for B in 1 16 64; do timeout 300 python bench.py --decode --batch $B --steps 20 --warmup 5 2>gpurun_out/decb_$B.err | tail -1; done > gpurun_out/decbench.jsonl
timeout 300 python bench.py --decode --batch 1 --wbits 3 --abits 3 --steps 20 --warmup 5 2>>gpurun_out/decb_1.err | tail -1 >> gpurun_out/decbench.jsonl
