#!/bin/bash
# Bench lines per library and order: tools/ab_orders.sh "1 2" lib1.so lib2.so ...
ORDERS=$1; shift
for lib in "$@"; do
  for K in $ORDERS; do
    FERMAT_B200_LIB=$lib python bench.py --order $K --steps 50 --warmup 3 --no-e2e --no-cpu-baseline ${AB_ARGS} 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$(basename $lib)', 'K=$K', 'fused_ms', round(d['ms_per_step'],4), 'fwd_ms', round(d['fwd']['ms_per_step'],4), 'frac', round(d['roofline']['frac'],4))"
  done
done
