#!/bin/bash
# Round-2 measurement call: tests, headline bench, per-order lines, ncu captures
# (full set + executed FP32 op counts) of the fused tile kernels at K = 1, 2, 3.
#   bash tools/r02_gpu.sh TAG [tests|notests] [orders...]
T=${1:-r02a}; TESTS=${2:-tests}; shift 2; ORDERS=${@:-"1 2 3"}
mkdir -p gpurun_out
O=gpurun_out/$T
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > ${O}_smi.txt
if [ "$TESTS" = tests ]; then
  timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > ${O}_pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > ${O}_smoke.log 2>&1
fi
timeout 600 python bench.py > ${O}_bench_k3.json 2> ${O}_bench_k3.err
for k in $ORDERS; do
  [ $k = 3 ] || timeout 600 python bench.py --order $k --no-e2e --no-cpu-baseline > ${O}_bench_k$k.json 2>> ${O}_bench.err
done
FL=smsp__sass_thread_inst_executed_op_fadd_pred_on.sum,smsp__sass_thread_inst_executed_op_fmul_pred_on.sum,smsp__sass_thread_inst_executed_op_ffma_pred_on.sum,smsp__sass_thread_inst_executed_op_fadd2_pred_on.sum,smsp__sass_thread_inst_executed_op_fmul2_pred_on.sum,smsp__sass_thread_inst_executed_op_ffma2_pred_on.sum
for k in $ORDERS; do
  CMD="python bench.py --order $k --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-gate"
  timeout 600 $CMD > ${O}_plain_k$k.log 2>&1 && \
  timeout 1200 ncu --set full --metrics $FL --clock-control none --import-source on -k regex:path_kernel -s 3 -c 1 \
    -o ${O}_fused_k$k $CMD > ${O}_ncu_k$k.log 2>&1
done
tail -3 ${O}_pytest_gpu.log 2>/dev/null; cat ${O}_smoke.log 2>/dev/null; for f in ${O}_bench_*.json; do echo "$f: $(head -c 400 $f)"; done
ls -la gpurun_out | tail -20
