# Round-2: look-back tickets + NCCL entry point tests, smoke
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_parity.py -x -q -m gpu -k "shard or chunked or long or ties or no_hist or hist" > gpurun_out/pytest_t.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
