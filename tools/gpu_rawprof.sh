set -x
timeout 300 ncu --set full --clock-control none -k regex:splitq_gemm2 -s 3 -c 1 -o gpurun_out/raw python tools/gemm_latency.py 16384x3584x3584 > gpurun_out/ncu_raw.log 2>&1; echo rc=$?
python tools/ncu_summary.py full gpurun_out/raw.ncu-rep gpurun_out/ncu_raw.json
ncu -i gpurun_out/raw.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip -9 > gpurun_out/raw_sass.csv.gz
rm -f gpurun_out/*.ncu-rep
