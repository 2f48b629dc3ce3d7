# K1 per-round barrier group size A/B (512 = default)
cp paper_2605_19929_b200/libsplitq_b200.so /tmp/def.so
for V in def sync256 sync1024; do
  if [ $V = def ]; then cp /tmp/def.so paper_2605_19929_b200/libsplitq_b200.so; else cp build/$V.so paper_2605_19929_b200/libsplitq_b200.so; fi
  for P in q; do echo "$V $(timeout 300 python tools/k1_prof.py --proj $P --tokens 65536 --iters 5 2>&1 | tail -1)"; done
done
cp /tmp/def.so paper_2605_19929_b200/libsplitq_b200.so
