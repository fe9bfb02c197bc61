mkdir -p gpurun_out
L=paper_2502_12665_b200/lib
for v in liba2ats liba2ats_nv64; do
  A2ATS_LIB=$L/$v.so timeout 300 python tools/kbench.py --config C4 --select-only --postings --iters 6 > gpurun_out/kb_c4s_$v.log 2>&1
  A2ATS_LIB=$L/$v.so timeout 300 python tools/kbench.py --config C4 --postings --no-append --iters 6 > gpurun_out/kb_c4_$v.log 2>&1
  A2ATS_LIB=$L/$v.so timeout 300 python tools/kbench.py --config C2 --no-append --iters 6 > gpurun_out/kb_c2_$v.log 2>&1
done
A2ATS_LIB=$L/liba2ats_phases_nv64.so timeout 300 python tools/timeline_probe.py --config C4 --postings --graph --iters 3 > gpurun_out/tl_nv64.log 2>&1
