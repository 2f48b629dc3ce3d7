# Round 2 check: every GPU test, the driver bench (and its variants), decode, config 5,
# then the launch list + ncu --set full of K1 and the split GEMM (profiles/r02)
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_r02.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu_r02.log
timeout 900 python bench.py > gpurun_out/bench_r02.log 2> gpurun_out/bench_r02.err; echo bench rc=$?
timeout 900 python bench.py --abits 8 --no-e2e --no-cpu-baseline --no-fp32-out > gpurun_out/bench_r02_w4a8.log 2>&1; echo w4a8 rc=$?
timeout 900 python bench.py --schedule serial --no-e2e --no-cpu-baseline --no-fp32-out > gpurun_out/bench_r02_serial.log 2>&1; echo serial rc=$?
timeout 600 python tools/bench_decode.py --specs 4:4 > gpurun_out/decode_r02.jsonl 2> gpurun_out/decode_r02.err; echo dec rc=$?
timeout 900 python tools/bench_c5.py > gpurun_out/c5_r02.json 2> gpurun_out/c5_r02.err; echo c5 rc=$?
bash tools/gpu_profile.sh r02
