mkdir -p gpurun_out
for pass in 1 2; do
for cfg in "1 2" "2 2" "2 3" "3 3"; do
  set -- $cfg
  timeout 300 python bench.py --steps 40 --no-cpu-baseline --e2e-lag $1 --stream-slots $2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('lag $1 slots $2 pass $pass', round(d['ms_per_step'],4), 'e2e', round(e['ms_per_step'],3), 'blocking', round(e['blocking']['ms_per_step'],3), 'link duplex', round(e['link']['duplex_ms'],3), 'frac', round(e['link']['frac'],3))"
done; done
