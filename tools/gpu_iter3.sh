mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/it_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/it_pytest.log
timeout 900 python tools/lut_sweep.py --out gpurun_out/lut_sweep.json > gpurun_out/lut_sweep.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"qprep|prep_kernel|select|attn|lut_fma" -c 60 --csv --log-file gpurun_out/launches_c4.csv python bench.py --config C4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_l4.log 2>&1
