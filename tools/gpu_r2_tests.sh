# Round-2: codebook-construction GPU tests
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_codebook.py -x -q -m gpu > gpurun_out/pytest_cb.log 2>&1
