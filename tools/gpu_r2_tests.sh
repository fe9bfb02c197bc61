# Round-2: two-CTAs-per-SM scan -- tests + C4 timing
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_r2.py tests/test_gpu_sharded.py tests/test_gpu_postings.py -x -q -m gpu -k "long or stream or c4 or C4 or select or shard or postings" > gpurun_out/pytest_scan.log 2>&1
timeout 300 python tools/kbench.py --config C4 --select-only --iters 8 > gpurun_out/sel_c4.log 2>&1
