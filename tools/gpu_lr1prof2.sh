# ncu --set full of the prefill LR1 launches (q projection, 65,536 tokens) + the final text-score lines
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none -k regex:splitq_gemm2 -s 3 -c 2 -o gpurun_out/lr1 python tools/k1_prof.py --proj q --tokens 65536 --iters 1 > gpurun_out/ncu_lr1.log 2>&1; echo ncu rc=$?
ncu -i gpurun_out/lr1.ncu-rep --page details --csv > gpurun_out/lr1_details.csv 2>&1
rm -f gpurun_out/lr1.ncu-rep
bash tools/gpu_tsprof.sh
