# Round profile: launch list of the bench step + ncu --set full of every kernel of one step.
# Usage (on the GPU box): bash tools/gpu_profile.sh <tag>
set -x
TAG=${1:-r01}
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $B > gpurun_out/ncu_launch_$TAG.log 2>&1; echo launches rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k1w -s 7 -c 7 -o gpurun_out/k1_$TAG $B > gpurun_out/ncu_k1_$TAG.log 2>&1; echo k1 rc=$?
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:splitq_gemm2 -s 21 -c 15 -o gpurun_out/gemm_$TAG $B > gpurun_out/ncu_gemm_$TAG.log 2>&1; echo gemm rc=$?
python tools/ncu_summary.py launches gpurun_out/launches_$TAG.csv gpurun_out/launches_$TAG.json
python tools/ncu_summary.py full gpurun_out/k1_$TAG.ncu-rep gpurun_out/ncu_k1_$TAG.json
python tools/ncu_summary.py full gpurun_out/gemm_$TAG.ncu-rep gpurun_out/ncu_gemm_$TAG.json
# keep the merge-back under the 64 MiB limit: summaries only (+ compressed source pages)
for r in k1 gemm; do
  ncu -i gpurun_out/${r}_$TAG.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip -9 > gpurun_out/${r}_${TAG}_sass.csv.gz
done
rm -f gpurun_out/*.ncu-rep
du -sh gpurun_out
