#!/bin/bash
# A/B timing of experimental libraries (build_variant) on the headline step:
#   tools/ab_libs.sh ORDER lib1.so lib2.so ...   (two alternating passes)
K=$1; shift
for pass in 1 2; do
  for lib in "$@"; do
    FERMAT_B200_LIB=$lib python bench.py --order $K --steps 50 --no-e2e --no-cpu-baseline 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$(basename $lib) pass $pass', round(d['ms_per_step'],4), 'fwd', round(d['fwd']['ms_per_step'],4), d['clocks']['sm_mhz'])"
  done
done
