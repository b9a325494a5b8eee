#!/bin/bash
# Round-2 measurement set: GPU tests, smoke, bench lines (every order, configs
# 1/3/4, reference arm), ncu launch list and full captures (fused K=1,2,3 with
# executed FP32 op counts; the config-3 order-3 enumeration kernel).
#   bash tools/r02_final.sh TAG [notests]
T=${1:-r02x}
mkdir -p gpurun_out
O=gpurun_out/$T
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > ${O}_smi.txt
if [ "$2" != notests ]; then
  timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -30 > ${O}_pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > ${O}_smoke.log 2>&1
fi
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
CMD="python bench.py --steps 3 --warmup 3 --no-gate"
timeout 600 $CMD > ${O}_plain_launch.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file ${O}_launches.csv $CMD > ${O}_ncu_launch.log 2>&1
FL=smsp__sass_thread_inst_executed_op_fadd_pred_on.sum,smsp__sass_thread_inst_executed_op_fmul_pred_on.sum,smsp__sass_thread_inst_executed_op_ffma_pred_on.sum,smsp__sass_thread_inst_executed_op_fadd2_pred_on.sum,smsp__sass_thread_inst_executed_op_fmul2_pred_on.sum,smsp__sass_thread_inst_executed_op_ffma2_pred_on.sum
for k in 1 2 3; do
  CMD="python bench.py --order $k --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-gate"
  timeout 600 $CMD > ${O}_plain_k$k.log 2>&1 && \
  timeout 1200 ncu --set full --metrics $FL --clock-control none --import-source on -k regex:path_kernel -s 3 -c 1 \
    -o ${O}_fused_k$k $CMD > ${O}_ncu_k$k.log 2>&1
done
CMD="python bench.py --workload config3 --alphabet walls --no-records --steps 1 --warmup 1"
timeout 600 $CMD > ${O}_plain_enum.log 2>&1 && \
  timeout 1200 ncu --set full --metrics $FL --clock-control none --import-source on -k regex:enum_kernel -s 5 -c 1 \
    -o ${O}_enum_k3 $CMD > ${O}_ncu_enum.log 2>&1
tail -3 ${O}_pytest_gpu.log 2>/dev/null; cat ${O}_smoke.log 2>/dev/null; for f in ${O}_bench_*.json; do echo "$f: $(head -c 300 $f)"; done
