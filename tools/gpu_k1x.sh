set -x
mkdir -p gpurun_out
for T in 8192 16384 32768; do for W in 0 8; do
SPLITQ_K1_WPR=$W timeout 600 python bench.py --no-e2e --no-cpu-baseline --tokens $T --steps 5 --warmup 3 --schedule serial > gpurun_out/k1x_${T}_$W.log 2>&1; echo rc=$?
done; done
