set -x
B="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:splitq_gemm2 -s 0 -c 3 -o gpurun_out/gq $B > gpurun_out/ncu_gq.log 2>&1; echo rc=$?
python tools/ncu_summary.py full gpurun_out/gq.ncu-rep gpurun_out/ncu_gq.json
ncu -i gpurun_out/gq.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip -9 > gpurun_out/gq_sass.csv.gz
rm -f gpurun_out/*.ncu-rep
