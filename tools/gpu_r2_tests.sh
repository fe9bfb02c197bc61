# Round-2: postings engine tests + timing
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_postings.py -x -q -m gpu > gpurun_out/pytest_post.log 2>&1
for cfg in C4 C2; do for e in "" "--postings"; do
  echo "== $cfg $e" >> gpurun_out/sel_eng.log
  timeout 300 python tools/kbench.py --config $cfg --select-only --iters 8 $e 2>&1 | tail -2 >> gpurun_out/sel_eng.log
done; done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"select_postings" -s 2 -c 1 -o gpurun_out/full_post_c4 -f python tools/kbench.py --config C4 --select-only --iters 4 --postings > gpurun_out/ncu_post.log 2>&1
