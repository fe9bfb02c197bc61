# quick iteration: long-context parity + select timing + timeline
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider > gpurun_out/it_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/it_pytest.log
timeout 120 python tools/kbench.py --config C4 --select-only --iters 6 > gpurun_out/it_kb.log 2>&1
timeout 120 python tools/kbench.py --config C4 --iters 4 >> gpurun_out/it_kb.log 2>&1
A2ATS_LIB=paper_2502_12665_b200/lib/liba2ats_phases.so timeout 300 python tools/timeline_probe.py --config C4 --select-only --iters 3 > gpurun_out/it_tl.log 2>&1
