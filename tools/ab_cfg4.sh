# A/B of the config-4 step time between two libraries: tools/ab_cfg4.sh libA libB [alphabet]
AL=${3:-walls}
for rep in 1 2; do for lib in "$1" "$2"; do
  FERMAT_B200_LIB=$lib timeout 600 python bench.py --workload config4 --alphabet $AL --steps 5 2>/dev/null \
    | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$lib', d['ms_per_step'])"
done; done
