# Round-2: ncu launch list + full capture (with source) of the C4 score+top-K kernels
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:"prefetch|qprep|prep_kernel|select" -c 20 --csv --log-file gpurun_out/launches_sel_c4.csv python tools/kbench.py --config C4 --select-only --iters 4 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"select_stream" -s 1 -c 1 -o gpurun_out/full_stream_c4 -f python tools/kbench.py --config C4 --select-only --iters 3 > gpurun_out/ncu_stream.log 2>&1
