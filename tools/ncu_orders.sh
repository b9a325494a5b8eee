# ncu --set full of one fused tile launch per order (bench.py --order K)
mkdir -p gpurun_out
for k in "$@"; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:path_kernel -s 2 -c 1 \
    -o gpurun_out/ncu_fused_k$k python bench.py --order $k --steps 1 --warmup 3 --no-e2e --no-cpu-baseline \
    > gpurun_out/ncu_fused_k$k.log 2>&1
done
