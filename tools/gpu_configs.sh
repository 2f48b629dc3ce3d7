# The BASELINE configs beyond the headline (each one bench line / decode lines)
set -x
mkdir -p gpurun_out
B="python bench.py --no-e2e --no-cpu-baseline"
timeout 600 $B --model 3b --tokens 4096 --steps 20 --warmup 5 > gpurun_out/cfg_c2.log 2>&1; echo rc=$?
timeout 600 $B --model 3b --tokens 65536 --steps 5 --warmup 3 > gpurun_out/cfg_c2_big.log 2>&1; echo rc=$?
timeout 600 $B --abits 8 --wbits 4 --steps 5 --warmup 3 > gpurun_out/cfg_c3_a8.log 2>&1; echo rc=$?
timeout 600 $B --tokens 8192 --abits 3 --wbits 3 --steps 20 --warmup 5 > gpurun_out/cfg_c4_w3a3.log 2>&1; echo rc=$?
timeout 600 $B --tokens 8192 --abits 2 --wbits 3 --steps 20 --warmup 5 > gpurun_out/cfg_c4_w3a2.log 2>&1; echo rc=$?
timeout 600 python tools/bench_decode.py --specs 4:4,3:3,3:2 > gpurun_out/decode_all.jsonl 2> gpurun_out/decode_all.err; echo rc=$?
timeout 1500 python tools/bench_c5.py > gpurun_out/c5.json 2> gpurun_out/c5.err; echo rc=$?
