#!/bin/bash
# Per-kernel durations (ncu launch list) of the K=3 fused + fwd steps for each library.
#   tools/ab_ncu.sh lib1.so lib2.so ...  -> gpurun_out/ab_ncu_<name>.csv + summary
for lib in "$@"; do
  name=$(basename $lib .so)
  FERMAT_B200_LIB=$lib ncu --metrics gpu__time_duration.sum --clock-control none -k regex:path_kernel -c 64 --csv \
    --log-file gpurun_out/ab_ncu_$name.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline ${AB_ARGS} > /dev/null 2>&1
  python tools/ncu_launch_summary.py gpurun_out/ab_ncu_$name.csv $name
done
