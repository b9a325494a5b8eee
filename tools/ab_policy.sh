#!/bin/bash
# Bench lines per kernel policy: tools/ab_policy.sh auto bucket tile ...
for pol in "$@"; do
  for rep in 1 2; do
    python bench.py --steps 50 --warmup 3 --no-e2e --no-cpu-baseline --policy $pol ${AB_ARGS} 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$pol', 'fused_ms', round(d['ms_per_step'],4), 'fwd_ms', round(d['fwd']['ms_per_step'],4), 'conv', d['converged_fraction'], 'frac', round(d['roofline']['frac'],4), 'launches', d['gpu_launches'], 'clk', d['clocks']['sm_mhz'])"
  done
done
