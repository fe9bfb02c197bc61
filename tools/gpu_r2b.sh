# Round-2 session 3: state check after restore -- GPU tests, smoke, C4 select engines, timelines
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 300 python tools/kbench.py --config C4 --select-only --iters 6 > gpurun_out/kb_scan.log 2>&1
timeout 300 python tools/kbench.py --config C4 --select-only --postings --iters 6 > gpurun_out/kb_post.log 2>&1
timeout 300 python tools/kbench.py --config C4 --iters 6 > gpurun_out/kb_step.log 2>&1
timeout 300 python tools/timeline_probe.py --config C4 --select-only --iters 3 > gpurun_out/tl_scan.log 2>&1
timeout 300 python tools/timeline_probe.py --config C4 --postings --iters 3 > gpurun_out/tl_post.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_sel.csv python tools/kbench.py --config C4 --select-only --postings --iters 4 > gpurun_out/ncu_ls.log 2>&1
timeout 1800 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
echo done
