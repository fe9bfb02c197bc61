mkdir -p gpurun_out
A2ATS_LIB=paper_2502_12665_b200/lib/liba2ats_phases.so timeout 300 python tools/timeline_probe.py --config C4 --select-only --iters 3 > gpurun_out/it_tl.log 2>&1
