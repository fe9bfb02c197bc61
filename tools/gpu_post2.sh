mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_deferred_encode.py -x -q -m gpu > gpurun_out/pytest_lag.log 2>&1
