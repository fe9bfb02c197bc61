./tools/gather_bench > gpurun_out/gather2.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu5.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu5.log
for v in liba2ats liba2ats_r128 liba2ats_r512 liba2ats_r1024; do echo "== $v" >> gpurun_out/kb5.log; A2ATS_LIB=paper_2502_12665_b200/lib/$v.so timeout 300 python tools/kbench.py --iters 4 >> gpurun_out/kb5.log 2>&1; done
echo "== C4 b16" >> gpurun_out/kb5.log; timeout 300 python tools/kbench.py --iters 3 --config C4 --batch 16 >> gpurun_out/kb5.log 2>&1
