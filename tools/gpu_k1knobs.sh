# K1 experiment knobs: L2 prefetch distance, warps per SM, PF / SYNC, on the q and down inputs
mkdir -p gpurun_out
run() { echo "== $*"; env "$@" timeout 300 python tools/k1_prof.py --proj $P --tokens 65536 --iters 5 2>&1 | tail -1; }
for P in q down; do
  run X=0
  run SPLITQ_K1_L2PF=1
  run SPLITQ_K1_L2PF=2
  run SPLITQ_K1_L2PF=4
done
P=q
run SPLITQ_K1_SYNC=0
run SPLITQ_K1_SYNC=0 SPLITQ_K1_L2PF=1
run SPLITQ_K1_SYNC=0 SPLITQ_K1_L2PF=2
P=down
for W in 12 16 20 24; do
  run SPLITQ_K1_WSM=$W
  run SPLITQ_K1_WSM=$W SPLITQ_K1_PF=1
done
run SPLITQ_K1_PF=1
run SPLITQ_K1_SYNC=1
