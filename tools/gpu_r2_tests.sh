# Round-2: scan ring depth (5 stages, single table) -- tests + C4 timing vs 4 stages
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_r2.py tests/test_gpu_sharded.py -x -q -m gpu -k "long or stream or c4 or C4 or select or shard" > gpurun_out/pytest_scan.log 2>&1
for v in liba2ats liba2ats_s4 liba2ats liba2ats_s4; do
  echo "== $v" >> gpurun_out/sel_ring.log
  A2ATS_LIB=paper_2502_12665_b200/lib/$v.so timeout 300 python tools/kbench.py --config C4 --select-only --iters 8 2>&1 | tail -3 >> gpurun_out/sel_ring.log
done
