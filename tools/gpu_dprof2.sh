# ncu --set full of the decode kernels (K1 + GEMV) of one projection at batch 1 and 8
set -x
mkdir -p gpurun_out
PROJ=${PROJ:-q}
for B in 1 8; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k1w|gv_kernel' -s 8 -c 4 \
  -o gpurun_out/dec_b$B python tools/decode_micro.py --proj $PROJ --batches $B --iters 2 > gpurun_out/ncu_dec_b$B.log 2>&1; echo ncu rc=$?
python tools/ncu_summary.py full gpurun_out/dec_b$B.ncu-rep gpurun_out/ncu_dec_b$B.json
ncu -i gpurun_out/dec_b$B.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/dec_b${B}_sass.csv.gz
done
