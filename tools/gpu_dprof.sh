set -x
timeout 300 ncu --set full --clock-control none -k regex:splitq_gemm2 -s 9 -c 3 -o gpurun_out/dq python tools/decode_micro.py --proj q --batches 64 --iters 2 > gpurun_out/ncu_dq.log 2>&1; echo rc=$?
python tools/ncu_summary.py full gpurun_out/dq.ncu-rep gpurun_out/ncu_dq.json
ncu -i gpurun_out/dq.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip -9 > gpurun_out/dq_sass.csv.gz
rm -f gpurun_out/*.ncu-rep
