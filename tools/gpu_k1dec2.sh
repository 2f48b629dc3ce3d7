# K1 change check: parity tests, prefill K1 times, decode bench line, decode phase clocks
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_k1w.py tests/test_gpu_forward.py -q -x > gpurun_out/k1d_pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/k1d_pytest.log
for P in q down; do timeout 300 python tools/k1_prof.py --proj $P --tokens 65536 --iters 5 2>&1 | tail -1; done
timeout 300 python bench.py --decode --batch 1 --steps 20 --warmup 5 2>/dev/null | tail -1 | cut -c 1-400
bash tools/gpu_k1trace2.sh | tail -4
