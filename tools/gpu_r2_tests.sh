# Round-2: codebook trainer timing, compute-sanitizer on small steps, full GPU suite + smoke
mkdir -p gpurun_out
timeout 600 python tools/train_bench.py > gpurun_out/train_r2.json 2> gpurun_out/train_r2.err
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_small.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitize_$tool.log
done
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
