#!/bin/bash
# A/B timing of experimental libraries (python -m paper_2510_16172_b200.build --variant ...):
#   tools/ab_time.sh lib1.so lib2.so ...   -> one bench line per library (K=3 fused step)
for lib in "$@"; do
  for rep in 1 2; do
    FERMAT_B200_LIB=$lib python bench.py --steps 50 --warmup 3 --no-e2e --no-cpu-baseline ${AB_ARGS} 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$lib', 'fused_ms', round(d['ms_per_step'],4), 'fwd_ms', round(d['fwd']['ms_per_step'],4), 'conv', d['converged_fraction'], 'frac', round(d['roofline']['frac'],4))"
  done
done
