mkdir -p gpurun_out
L=paper_2502_12665_b200/lib
for v in liba2ats liba2ats_npf; do
  A2ATS_LIB=$L/$v.so timeout 300 python tools/kbench.py --config C4 --select-only --postings --iters 8 > gpurun_out/kb_post_$v.log 2>&1
done
for v in liba2ats_phases liba2ats_phases_npf; do
  A2ATS_LIB=$L/$v.so timeout 300 python tools/timeline_probe.py --config C4 --postings --iters 3 > gpurun_out/tl_post_$v.log 2>&1
done
