# round-end check: smoke, all GPU tests, default bench, reference arm
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
s0=$(date +%s); timeout 900 python bench.py > gpurun_out/bench_default.log 2> gpurun_out/bench_default.err; echo bench rc=$? secs=$(( $(date +%s) - s0 ))
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo ref rc=$?
