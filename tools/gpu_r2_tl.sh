# Round-2: per-CTA timeline of C4 score+top-K + ncu launch list of the same
mkdir -p gpurun_out
for pf in 0 12; do
  echo "== prefetch $pf" >> gpurun_out/tl_c4.log
  A2ATS_L2_PREFETCH=$pf timeout 300 python tools/timeline_probe.py --config C4 --select-only --iters 4 >> gpurun_out/tl_c4.log 2>&1
done
A2ATS_L2_PREFETCH=0 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct --clock-control none -c 40 --csv --log-file gpurun_out/launches_sel_c4_pf0.csv python tools/kbench.py --config C4 --select-only --iters 4 > /dev/null 2>&1
A2ATS_L2_PREFETCH=12 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct --clock-control none -c 40 --csv --log-file gpurun_out/launches_sel_c4_pf12.csv python tools/kbench.py --config C4 --select-only --iters 4 > /dev/null 2>&1
