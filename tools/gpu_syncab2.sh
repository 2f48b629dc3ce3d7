# K1: CTA barrier every round (default) vs every 2nd / 4th round
cp paper_2605_19929_b200/libsplitq_b200.so /tmp/def.so
for V in def sync_every2 sync_every4; do
  if [ $V = def ]; then cp /tmp/def.so paper_2605_19929_b200/libsplitq_b200.so; else cp build/$V.so paper_2605_19929_b200/libsplitq_b200.so; fi
  echo "$V $(timeout 300 python tools/k1_prof.py --proj q --tokens 65536 --iters 5 2>&1 | tail -1)"
done
cp /tmp/def.so paper_2605_19929_b200/libsplitq_b200.so
