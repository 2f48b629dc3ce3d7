# GEMV change check: decode parity tests, decode bench lines, the gate GEMV alone (ncu duration)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_forward.py tests/test_gpu_memsafety.py -q -x 2>&1 | tail -2
for B in 1 16; do timeout 300 python bench.py --decode --batch $B --steps 30 --warmup 5 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("decode B", d["config"]["batch"], round(d["ms_per_step"]*1e3,1), "us")'; done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:gv_kernel -s 4 -c 1 python tools/decode_micro.py --proj gate --batches 1 --iters 2 2>&1 | grep -E "gpu__time|dram__bytes"
