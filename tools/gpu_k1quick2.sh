# K1 change check: K1 / forward parity tests, then K1 time on the q and down inputs
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_k1w.py tests/test_gpu_forward.py tests/test_gpu_fullsize.py -q -x > gpurun_out/k1q_pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/k1q_pytest.log
for P in q down; do timeout 300 python tools/k1_prof.py --proj $P --tokens 65536 --iters 5 2>&1 | tail -1; done
for P in q; do timeout 300 python tools/k1_prof.py --proj $P --tokens 65536 --iters 5 --abits 8 2>&1 | tail -1; done
