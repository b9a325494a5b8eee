set -x; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/r01i_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r01i_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/r01i_bench_k3.json 2> gpurun_out/r01i_bench_k3.err
tail -3 gpurun_out/r01i_pytest_gpu.log; cat gpurun_out/r01i_smoke.log; cat gpurun_out/r01i_bench_k3.json
