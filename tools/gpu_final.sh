# Round measurement set: tests, smoke, bench lines (every order, configs 1/3/4,
# reference arm), ncu launch list and one full capture of the K=3 fused kernel.
# usage: bash tools/gpu_final.sh TAG   (outputs gpurun_out/TAG_*)
T=${1:-r01i}
mkdir -p gpurun_out
O=gpurun_out/$T
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > ${O}_smi.txt
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -5 > ${O}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > ${O}_smoke.log 2>&1
timeout 600 python bench.py > ${O}_bench_k3.json 2> ${O}_bench_k3.err
for k in 1 2 4 5; do
  timeout 600 python bench.py --order $k --no-e2e > ${O}_bench_k$k.json 2>> ${O}_bench.err
done
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > ${O}_bench_ref.json 2>> ${O}_bench.err
timeout 900 python bench.py --workload config1 --steps 10 > ${O}_bench_cfg1.json 2>> ${O}_bench.err
timeout 900 python bench.py --workload config3 --alphabet walls --visibility --steps 5 > ${O}_bench_cfg3w.json 2>> ${O}_bench.err
timeout 1200 python bench.py --workload config3 --alphabet all --steps 3 > ${O}_bench_cfg3a.json 2>> ${O}_bench.err
timeout 900 python bench.py --workload config4 --alphabet walls --steps 5 > ${O}_bench_cfg4w.json 2>> ${O}_bench.err
timeout 900 python bench.py --workload config4 --alphabet all --steps 2 > ${O}_bench_cfg4a.json 2>> ${O}_bench.err
timeout 900 python tools/f64_rate.py > ${O}_f64_rate.txt 2>> ${O}_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file ${O}_launches.csv python bench.py --steps 3 --warmup 3 > ${O}_ncu_launch.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:path_kernel -s 2 -c 1 \
  -o ${O}_fused_k3 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > ${O}_ncu_full.log 2>&1
tail -2 ${O}_pytest_gpu.log; cat ${O}_smoke.log; for f in ${O}_bench_*.json; do echo "$f: $(head -c 300 $f)"; done
