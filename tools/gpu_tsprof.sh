# ncu --set full of one text-score launch (source lines), summarised by tools/ncu_lines.py
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:text_score -c 1 -o gpurun_out/ts python tools/ts_micro.py --channels 296 --iters 1 > gpurun_out/ncu_ts.log 2>&1; echo ncu rc=$?
python tools/ncu_lines.py gpurun_out/ts.ncu-rep 45 > gpurun_out/tslines.txt 2>&1
ncu -i gpurun_out/ts.ncu-rep --page details --csv > gpurun_out/ts_details.csv 2>&1
rm -f gpurun_out/ts.ncu-rep
