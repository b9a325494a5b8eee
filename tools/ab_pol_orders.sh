#!/bin/bash
# Bench lines per (policy, order): tools/ab_pol_orders.sh "4 5" tile bucket
ORDERS=$1; shift
for pol in "$@"; do
  for K in $ORDERS; do
    python bench.py --order $K --steps 50 --warmup 3 --no-e2e --no-cpu-baseline --policy $pol ${AB_ARGS} 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$pol', 'K=$K', 'fused_ms', round(d['ms_per_step'],4), 'fwd_ms', round(d['fwd']['ms_per_step'],4), 'frac', round(d['roofline']['frac'],4), 'launches', d['gpu_launches'])"
  done
done
