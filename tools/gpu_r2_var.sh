# Round-2: C4 score+top-K time of stream-kernel tuning variants (results of stripped variants are wrong by design)
mkdir -p gpurun_out
for pf in 0 12; do
for v in liba2ats liba2ats_ah0 liba2ats_ah8 liba2ats_none liba2ats_none8; do
  echo "== $v pf $pf" >> gpurun_out/var_c4.log
  A2ATS_L2_PREFETCH=$pf A2ATS_LIB=paper_2502_12665_b200/lib/$v.so timeout 300 python tools/kbench.py --config C4 --select-only --iters 6 2>&1 | tail -2 >> gpurun_out/var_c4.log
done
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:"prefetch|select_stream" -c 6 --csv --log-file gpurun_out/launches_pf.csv python tools/kbench.py --config C4 --select-only --iters 3 > /dev/null 2>&1
