# decode step vs the LR1 GEMV K split (SPLITQ_GV_KSPLIT forces it)
for K in 0 2 4 8; do
  if [ $K = 0 ]; then E=""; else E="SPLITQ_GV_KSPLIT=$K"; fi
  for B in 1 16; do
    echo "ksplit=$K B=$B $(env $E timeout 300 python bench.py --decode --batch $B --steps 30 --warmup 5 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"]*1e3,1), "us")')"
  done
done
