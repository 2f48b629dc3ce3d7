# Round-2 final check (after the late K1 / MOCD / decode-bench commits): every GPU
# test, smoke, the driver bench and its variants, decode lines, config 5, then the
# launch list + ncu --set full of K1 and the split GEMM (profiles/r02c)
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_r02c.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu_r02c.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02c.log 2>&1; echo smoke rc=$?
timeout 900 python bench.py > gpurun_out/bench_r02c.log 2> gpurun_out/bench_r02c.err; echo bench rc=$?
timeout 900 python bench.py --abits 8 --no-e2e --no-cpu-baseline --no-fp32-out > gpurun_out/bench_r02c_w4a8.log 2>&1; echo w4a8 rc=$?
timeout 900 python bench.py --wbits 3 --abits 2 --no-e2e --no-cpu-baseline --no-fp32-out > gpurun_out/bench_r02c_w3a2.log 2>&1; echo w3a2 rc=$?
for B in 1 8 16 64; do timeout 300 python bench.py --decode --batch $B --steps 20 --warmup 5 2>/dev/null | tail -1; done > gpurun_out/decode_bench_r02c.jsonl; echo dec rc=$?
timeout 300 python bench.py --decode --batch 1 --wbits 3 --abits 3 --steps 20 --warmup 5 2>/dev/null | tail -1 >> gpurun_out/decode_bench_r02c.jsonl
timeout 300 python bench.py --decode --batch 1 --wbits 3 --abits 2 --steps 20 --warmup 5 2>/dev/null | tail -1 >> gpurun_out/decode_bench_r02c.jsonl
timeout 900 python tools/bench_c5.py > gpurun_out/c5_r02c.json 2> gpurun_out/c5_r02c.err; echo c5 rc=$?
bash tools/gpu_profile.sh r02c
