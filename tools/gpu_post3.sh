mkdir -p gpurun_out
L=paper_2502_12665_b200/lib
for v in liba2ats_phases_ns liba2ats_phases_t2; do
  A2ATS_LIB=$L/$v.so timeout 300 python tools/timeline_probe.py --config C4 --postings --iters 3 > gpurun_out/tl_post_$v.log 2>&1
done
