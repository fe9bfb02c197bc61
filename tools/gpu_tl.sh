mkdir -p gpurun_out
A2ATS_LIB=paper_2502_12665_b200/lib/liba2ats_phases.so timeout 300 python tools/timeline_probe.py --config C4 --iters 3 > gpurun_out/it_tl_step.log 2>&1
A2ATS_LIB=paper_2502_12665_b200/lib/liba2ats_phases.so timeout 300 python tools/timeline_probe.py --config C2 --iters 3 > gpurun_out/it_tl_c2.log 2>&1
