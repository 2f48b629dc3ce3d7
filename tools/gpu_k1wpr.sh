# K1 down input at 65,536 rows: warp rows (default) vs row groups of 2 / 4 / 8 warps
for W in 0 2 4 8; do
  if [ $W = 0 ]; then E=""; else E="SPLITQ_K1_WPR=$W"; fi
  echo "wpr=$W $(env $E timeout 300 python tools/k1_prof.py --proj down --tokens 65536 --iters 5 2>&1 | tail -1)"
done
for W in 2 4; do
  echo "wpr=$W q $(env SPLITQ_K1_WPR=$W timeout 300 python tools/k1_prof.py --proj q --tokens 65536 --iters 5 2>&1 | tail -1)"
done
