mkdir -p gpurun_out
export A2ATS_LIB=paper_2502_12665_b200/lib/liba2ats_phases.so
timeout 300 python tools/timeline_probe.py --config C4 --select-only --iters 4 > gpurun_out/tl_c4_sel.log 2>&1
timeout 300 python tools/timeline_probe.py --config C4 --iters 3 > gpurun_out/tl_c4_step.log 2>&1
timeout 300 python tools/timeline_probe.py --config C2 --select-only --iters 4 > gpurun_out/tl_c2_sel.log 2>&1
unset A2ATS_LIB
timeout 300 python tools/kbench.py --config C4 --select-only --iters 6 > gpurun_out/kb_c4_sel.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:select_stream -c 1 -s 2 -o gpurun_out/sel_c4 python tools/kbench.py --config C4 --select-only --iters 4 > gpurun_out/ncu_sel_c4.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:prep_kernel -c 1 -s 2 -o gpurun_out/prep_c4 python tools/kbench.py --config C4 --select-only --iters 4 > gpurun_out/ncu_prep_c4.log 2>&1
