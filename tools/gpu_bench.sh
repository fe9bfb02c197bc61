mkdir -p gpurun_out
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 900 python bench.py --no-cpu-baseline --a0 fused > gpurun_out/bench_c4_fused.json 2> gpurun_out/bench_c4_fused.err
timeout 600 python bench.py --config C2 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 600 python bench.py --config C2 --no-cpu-baseline --a0 fused > gpurun_out/bench_c2_fused.json 2> gpurun_out/bench_c2_fused.err
