mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/it_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/it_pytest.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/b2.json 2>gpurun_out/b2.err
timeout 300 python bench.py --config C4 --steps 10 --warmup 4 --no-cpu-baseline > gpurun_out/b4.json 2>gpurun_out/b4.err
A2ATS_LIB=paper_2502_12665_b200/lib/liba2ats_phases.so timeout 300 python tools/timeline_probe.py --config C4 --iters 3 > gpurun_out/it_tl_step.log 2>&1
