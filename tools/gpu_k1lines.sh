# K1 source-line attribution: ncu --set full of one q-type and one down K1 launch,
# then per-CUDA-line instruction counts / stall samples (tools/ncu_lines.py)
set -x
mkdir -p gpurun_out
for P in q down; do
  timeout 600 python tools/k1_prof.py --proj $P --tokens 65536 --iters 1 > gpurun_out/k1prof_$P.log 2>&1; echo plain rc=$?
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1w -s 2 -c 1 -o gpurun_out/k1l_$P python tools/k1_prof.py --proj $P --tokens 65536 --iters 1 > gpurun_out/ncu_k1l_$P.log 2>&1; echo ncu rc=$?
  python tools/ncu_lines.py gpurun_out/k1l_$P.ncu-rep 80 > gpurun_out/k1lines_$P.txt 2>&1
  ncu -i gpurun_out/k1l_$P.ncu-rep --page source --csv --print-source cuda,sass 2>/dev/null | gzip -9 > gpurun_out/k1l_${P}_src.csv.gz
  ncu -i gpurun_out/k1l_$P.ncu-rep --page details --csv > gpurun_out/k1l_${P}_details.csv 2>&1
  rm -f gpurun_out/k1l_$P.ncu-rep
done
