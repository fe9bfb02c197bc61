mkdir -p gpurun_out
timeout 300 python tools/timeline_probe.py --config C4 --postings --graph --iters 3 > gpurun_out/tl_post.log 2>&1
