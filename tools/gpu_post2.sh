mkdir -p gpurun_out
python tools/dbg/ph_dbg.py > gpurun_out/dbg.log 2>&1
timeout 900 python -m pytest tests/test_gpu_postings.py tests/test_gpu_codes8.py tests/test_gpu_per_head.py tests/test_gpu_deferred_encode.py -x -q -m gpu > gpurun_out/pytest_post.log 2>&1
