# bench line per order (device step, fused + fwd, roofline), two runs each
for k in ${ORDERS:-1 2 3 4 5}; do for rep in 1 2; do
  timeout 300 python bench.py --order $k --steps 50 --no-e2e --no-cpu-baseline 2>/dev/null \
   | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('K=$k', round(d['ms_per_step'],4), round(d['fwd']['ms_per_step'],4), round(d['roofline']['frac'],3))"
done; done
