# ncu full capture of the C4 select-only path with postings (qprep, LUT prep kernel, postings select)
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"qprep|prep_kernel|select_postings" -s 9 -c 3 -o gpurun_out/full_post -f python tools/kbench.py --config C4 --select-only --postings --iters 5 > gpurun_out/ncu_fp.log 2>&1
