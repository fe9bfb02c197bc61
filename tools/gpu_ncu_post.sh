# ncu full capture of the C4 select-only path with postings (LUT prep kernel, postings select, index build)
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"prep_kernel|select_postings|postings_build" -s 3 -c 4 -o gpurun_out/full_post2 -f python tools/kbench.py --config C4 --select-only --postings --iters 4 > gpurun_out/ncu_fp.log 2>&1
