# K1 wide-code (W4A8) change: K1 parity tests, then the q / down K1 at A4 and A8
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_k1w.py tests/test_gpu_forward.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -2
for A in 4 8; do for P in q down; do echo "A$A $(timeout 300 python tools/k1_prof.py --proj $P --tokens 65536 --iters 5 --abits $A 2>&1 | tail -1)"; done; done
