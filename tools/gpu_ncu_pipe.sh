mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:select_scan -c 1 -s 2 -o gpurun_out/pipe_c4 -f python tools/kbench.py --config C4 --select-only --iters 4 > gpurun_out/ncu_pipe.log 2>&1
