mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_r02a.log 2> gpurun_out/bench_r02a.err; echo bench rc=$?
tail -c 3500 gpurun_out/bench_r02a.log
timeout 900 python tools/bench_c5.py > gpurun_out/c5_r02a.log 2> gpurun_out/c5_r02a.err; echo c5 rc=$?
tail -c 1500 gpurun_out/c5_r02a.log; tail -5 gpurun_out/c5_r02a.err
