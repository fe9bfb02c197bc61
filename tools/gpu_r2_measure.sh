# Round-2 measurement: tests touched by the sharded changes, sharded C4 line at N = 1,
# the ncu launch list of the default bench command and a full capture of the C4 step kernels
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_parity_r2.py -x -q -m gpu > gpurun_out/pytest_sh.log 2>&1
timeout 900 python bench.py --sharded --no-cpu-baseline > gpurun_out/bench_c4_sharded1.json 2> gpurun_out/bench_c4_sharded1.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"qprep|prep_kernel|select|attn|lut_fma|stage_rows|combine|shard_state" -c 60 --csv --log-file gpurun_out/launches_c4.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_l4.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"qprep|prep_kernel|select_thresh|select_scan|attn" -s 15 -c 5 -o gpurun_out/full_c4 -f python tools/kbench.py --config C4 --iters 5 > gpurun_out/ncu_f4.log 2>&1
