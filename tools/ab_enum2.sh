#!/bin/bash
# A/B of two libraries on the enumeration workloads (configs 3 and 4), two alternating passes:
#   bash tools/ab_enum2.sh libA.so libB.so
LIBS=("$@")
for pass in 1 2; do
  for lib in "${LIBS[@]}"; do
    for wl in "config3 walls 10" "config3 all 3" "config4 walls 5"; do
      read -r W A S <<< "$wl"
      FERMAT_B200_LIB=$lib timeout 300 python bench.py --workload $W --alphabet $A --steps $S --warmup 3 \
        --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$(basename $lib) $W $A pass $pass', round(d['ms_per_step'],3), d.get('valid_paths'), d['clocks']['sm_mhz'])"
    done
  done
done
