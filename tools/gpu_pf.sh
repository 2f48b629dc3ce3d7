set -x
mkdir -p gpurun_out
timeout 500 python -m pytest tests/test_gpu_k1w.py tests/test_gpu_forward.py -x -q > gpurun_out/pytest_pf.log 2>&1; rc=$?; echo rc=$rc
[ $rc -eq 0 ] || exit 1
for T in 8192 16384; do for P in 0 1; do
SPLITQ_K1_PF=$P timeout 600 python bench.py --no-e2e --no-cpu-baseline --tokens $T --steps 5 --warmup 3 --schedule serial > gpurun_out/pf_${T}_$P.log 2>&1; echo rc=$?
done; done
timeout 600 python bench.py --no-e2e --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/pf_def.log 2>&1; echo rc=$?
