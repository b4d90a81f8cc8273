mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "two_kernel_dims or grouped_training" 2>&1 | tail -15 > gpurun_out/t1_pytest.log
