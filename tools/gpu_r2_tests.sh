# Round-2: new parity tests + smoke + full GPU suite
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity_r2.py -x -q -m gpu > gpurun_out/pytest_r2.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
