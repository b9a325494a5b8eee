# host-buffer pipeline: bitwise test, chunk/depth sweep (batched vs single copies)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_vjp.py -m gpu -x -q 2>&1 | tail -3 > gpurun_out/e2e_pytest.log
timeout 900 python tools/e2e_sweep.py > gpurun_out/e2e_sweep.log 2>&1
FP_E2E_SINGLE_COPIES=1 timeout 900 python tools/e2e_sweep.py > gpurun_out/e2e_sweep_single.log 2>&1
cat gpurun_out/e2e_pytest.log; paste gpurun_out/e2e_sweep.log gpurun_out/e2e_sweep_single.log
