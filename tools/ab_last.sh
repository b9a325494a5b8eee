#!/bin/bash
# A/B of two full libraries: bitwise outputs (fused, orders 1-3 and 9-64) and
# timing (fused orders 1-5, config-3 walls enumeration, long paths).
#   bash tools/ab_last.sh base.so new.so TAG
A=$1; B=$2; T=${3:-ab}
mkdir -p gpurun_out
O=gpurun_out/$T
python tools/ab_bits.py $A $B 1,2,3 > ${O}_bits.txt 2>&1
python tools/ab_wide.py $A $B > ${O}_wide.txt 2>&1
for k in 1 2 3 4 5; do bash tools/ab_libs.sh $k $A $B; done > ${O}_time.txt 2>&1
for pass in 1 2; do
  for lib in $A $B; do
    FERMAT_B200_LIB=$lib timeout 300 python bench.py --workload config3 --alphabet walls --steps 10 --warmup 3 \
      --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$(basename $lib) walls pass $pass', round(d['ms_per_step'],3), d['valid_paths'], d['clocks']['sm_mhz'])"
  done
done > ${O}_enum.txt 2>&1
cat ${O}_bits.txt ${O}_wide.txt ${O}_time.txt ${O}_enum.txt
