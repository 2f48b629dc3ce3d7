mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_r02b.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu_r02b.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"; echo smoke rc=$?
timeout 900 python bench.py > gpurun_out/bench_r02b.log 2> gpurun_out/bench_r02b.err; echo bench rc=$?
cat gpurun_out/bench_r02b.log | head -c 1500
