# W4A8 K1 A/B: build/head.so vs build/new.so
for V in head new; do cp build/$V.so paper_2605_19929_b200/libsplitq_b200.so
  for P in q down; do echo "$V A8 $(timeout 300 python tools/k1_prof.py --proj $P --tokens 65536 --iters 5 --abits 8 2>&1 | tail -1)"; done; done
