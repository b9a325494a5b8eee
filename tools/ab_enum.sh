set -e
mkdir -p gpurun_out
for pass in 1 2; do
 for lib in ablib/enum4.so ablib/enum3.so ablib/enum2.so; do
  for alpha in walls all; do
   st=10; [ $alpha = all ] && st=3
   FERMAT_B200_LIB=$lib timeout 300 python bench.py --workload config3 --alphabet $alpha --steps $st --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib $alpha pass $pass', round(d['ms_per_step'],3), d['valid_paths'], d['clocks']['sm_mhz'])"
  done
 done
done
