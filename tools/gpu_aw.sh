mkdir -p gpurun_out
for v in liba2ats liba2ats_aw4; do
  echo "== $v" >> gpurun_out/aw.log
  for c in C2 C4; do
  A2ATS_LIB=paper_2502_12665_b200/lib/$v.so timeout 300 python bench.py --config $c --steps 10 --warmup 4 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c', round(d['ms_per_step']*1e3,1), 'us/step', 'attn', round(d['kernels']['attention']['ms']*1e3,1), 'frac', round(d['roofline']['frac'],3))" >> gpurun_out/aw.log 2>&1
  done
done
A2ATS_LIB=paper_2502_12665_b200/lib/liba2ats_aw4.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "c1 or multi_tile or long_context or c4_full or needle or degenerate" >> gpurun_out/aw.log 2>&1
