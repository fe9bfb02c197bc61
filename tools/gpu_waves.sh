mkdir -p gpurun_out
for v in liba2ats liba2ats_w2 liba2ats_w4 liba2ats_w16; do
  echo "== $v" >> gpurun_out/waves.log
  for c in C2 C4; do
  A2ATS_LIB=paper_2502_12665_b200/lib/$v.so timeout 300 python bench.py --config $c --steps 10 --warmup 4 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c', round(d['ms_per_step']*1e3,1), 'us/step', 'prep', round(d['kernels']['prep']['ms']*1e3,1), 'sel', round(d['kernels']['select']['ms']*1e3,1), 'scoring', round(d['scoring']['ms']*1e3,1))" >> gpurun_out/waves.log 2>&1
  done
done
