mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_codes8.py tests/test_gpu_postings.py tests/test_gpu_per_head.py -x -q -m gpu > gpurun_out/pytest_c8.log 2>&1
