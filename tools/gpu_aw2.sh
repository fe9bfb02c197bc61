mkdir -p gpurun_out
for v in liba2ats liba2ats_n4s1 liba2ats_n4s2 liba2ats_n4s3; do
  A2ATS_LIB=paper_2502_12665_b200/lib/$v.so timeout 300 python bench.py --config C2 --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v C2', round(d['ms_per_step']*1e3,1), 'us/step', 'attn', round(d['kernels']['attention']['ms']*1e3,1))" >> gpurun_out/aw2.log 2>&1
done
