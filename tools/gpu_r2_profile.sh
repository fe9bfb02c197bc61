# Round-2 final profiles: ncu launch list of the default bench command (C4, posting-list engine),
# a full capture of the C4 step kernels (postings step) and of the index build
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"qprep|prep_kernel|lut_persist|select|attn|stage_rows|postings_build|head_" -c 120 --csv --log-file gpurun_out/launches_c4.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_l4.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"qprep|lut_persist|prep_kernel|select_postings|attn" -s 10 -c 5 -o gpurun_out/full_c4 -f python tools/kbench.py --config C4 --postings --iters 4 > gpurun_out/ncu_f4.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"postings_build" -s 1 -c 1 -o gpurun_out/full_build -f python tools/kbench.py --config C4 --select-only --postings --iters 1 > gpurun_out/ncu_fb.log 2>&1
