# Round-2 iteration: GPU tests + C4 score+top-K timing vs L2 warm-up depth + C4 bench line
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
for w in 0 10 14 18 22; do
  echo "== warm $w" >> gpurun_out/sel_c4.log
  A2ATS_L2_WARM=$w timeout 300 python tools/kbench.py --config C4 --select-only --iters 8 2>&1 | tail -3 >> gpurun_out/sel_c4.log
done
timeout 300 python bench.py --config C4 --steps 10 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
