mkdir -p gpurun_out
timeout 300 python tools/kbench.py --config C4 --select-only --postings --iters 6 > gpurun_out/kb_post.log 2>&1
timeout 300 python tools/timeline_probe.py --config C4 --postings --graph --iters 3 > gpurun_out/tl_post.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity_r2.py tests/test_gpu_postings.py -x -q -m gpu > gpurun_out/pytest_post.log 2>&1
