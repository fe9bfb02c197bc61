# Round-end measurement: bench lines, reference arm, launch lists, full ncu captures, tests, smoke
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 600 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 600 python bench.py --config C4 --steps 10 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 900 python bench.py --config C3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 python bench.py --sharded --steps 5 --warmup 3 > gpurun_out/bench_sharded1.json 2> gpurun_out/bench_sharded1.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"qprep|prep_kernel|select|attn|lut_fma" -c 80 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_l2.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"qprep|prep_kernel|select|attn|lut_fma" -c 60 --csv --log-file gpurun_out/launches_c4.csv python bench.py --config C4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_l4.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"prep_kernel|select_kernel|attn" -s 12 -c 3 -o gpurun_out/full_c2 -f python tools/kbench.py --config C2 --iters 6 > gpurun_out/ncu_f2.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"qprep|prep_kernel|select_thresh|select_scan|attn" -s 25 -c 5 -o gpurun_out/full_c4 -f python tools/kbench.py --config C4 --iters 7 > gpurun_out/ncu_f4.log 2>&1
