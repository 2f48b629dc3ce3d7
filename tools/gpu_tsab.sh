# text-score A/B: build/old.so vs the in-tree library on synthetic rank counts, then the MOCD parity tests
mkdir -p gpurun_out
cp paper_2605_19929_b200/libsplitq_b200.so /tmp/new.so
cp build/old.so paper_2605_19929_b200/libsplitq_b200.so
echo old; timeout 600 python tools/ts_micro.py --channels 592 --iters 2; timeout 300 python tools/ts_micro.py --n-cand 3548 --channels 592 --iters 2
cp /tmp/new.so paper_2605_19929_b200/libsplitq_b200.so
echo new; timeout 600 python tools/ts_micro.py --channels 592 --iters 2; timeout 300 python tools/ts_micro.py --n-cand 3548 --channels 592 --iters 2
timeout 900 python -m pytest tests/test_gpu_mocd.py tests/test_gpu_mocd_c5.py -q -x 2>&1 | tail -2
