# Round measurement: full GPU test suite, smoke, every path once (tools/sanitize_small.py), the bench
# lines (C4 default + engine / a0 variants, C2, C3, sharded at one rank, reference arm), ncu launch
# lists of the C4 and C2 bench commands and full captures of the C4 step kernels and the index build
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python tools/sanitize_small.py > gpurun_out/paths.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 900 python bench.py --no-cpu-baseline --engine scan > gpurun_out/bench_c4_scan.json 2> gpurun_out/bench_c4_scan.err
timeout 900 python bench.py --no-cpu-baseline --a0 fused > gpurun_out/bench_c4_fused.json 2> gpurun_out/bench_c4_fused.err
timeout 600 python bench.py --config C2 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 900 python bench.py --config C3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 900 python bench.py --sharded --no-cpu-baseline > gpurun_out/bench_c4_sharded1.json 2> gpurun_out/bench_c4_sharded1.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"qprep|prep_kernel|lut_persist|lut_fma|select|attn|stage_rows|postings_build|head_" -c 150 --csv --log-file gpurun_out/launches_c4.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_l4.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"qprep|prep_kernel|lut_persist|lut_fma|select|attn|stage_rows" -c 150 --csv --log-file gpurun_out/launches_c2.csv python bench.py --config C2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_l2.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"qprep|lut_persist|prep_kernel|select_postings|attn" -s 10 -c 5 -o gpurun_out/full_c4 -f python tools/kbench.py --config C4 --postings --no-append --iters 4 > gpurun_out/ncu_f4.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"postings_build" -s 1 -c 1 -o gpurun_out/full_build -f python tools/kbench.py --config C4 --select-only --postings --iters 1 > gpurun_out/ncu_fb.log 2>&1
