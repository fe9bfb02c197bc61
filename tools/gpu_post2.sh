mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_per_head.py -x -q -m gpu > gpurun_out/pytest_ph.log 2>&1
