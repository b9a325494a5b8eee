# A/B: streaming tile kernel vs one CTA per tile (FP_NO_STREAM_KERNEL=1), bench lines per order
for k in ${ORDERS:-3}; do for rep in 1 2; do for off in 0 1; do
  FP_NO_STREAM_KERNEL=$off timeout 300 python bench.py --order $k --steps 50 --no-e2e --no-cpu-baseline 2>/dev/null \
   | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('K=$k no_stream=$off', round(d['ms_per_step'],4), round(d['fwd']['ms_per_step'],4), round(d['roofline']['frac'],3))"
done; done; done
