mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_postings.py tests/test_gpu_parity_r2.py -x -q -m gpu > gpurun_out/pytest_post.log 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 600 python bench.py --config C2 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"select_postings|postings_build" -c 3 -o gpurun_out/full_post3 -f python tools/kbench.py --config C4 --select-only --postings --iters 3 > gpurun_out/ncu_fp.log 2>&1
