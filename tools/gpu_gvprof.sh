# ncu --set full of the gate-projection decode GEMV (batch 1): what bounds the weight stream
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'gv_kernel' -s 4 -c 1 -o gpurun_out/gv python tools/decode_micro.py --proj gate --batches 1 --iters 2 > gpurun_out/ncu_gv.log 2>&1; echo ncu rc=$?
python tools/ncu_lines.py gpurun_out/gv.ncu-rep 30 > gpurun_out/gvlines.txt 2>&1
ncu -i gpurun_out/gv.ncu-rep --page details --csv > gpurun_out/gv_details.csv 2>&1
ncu -i gpurun_out/gv.ncu-rep --page raw --csv > gpurun_out/gv_raw.csv 2>&1
rm -f gpurun_out/gv.ncu-rep
