mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "lut_engine or c1 or group" > gpurun_out/it_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/it_pytest.log
timeout 900 python tools/lut_sweep.py --out gpurun_out/lut_sweep.json > gpurun_out/lut_sweep.log 2>&1
