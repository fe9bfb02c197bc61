mkdir -p gpurun_out
for v in liba2ats liba2ats_s2 liba2ats_s3 liba2ats_s4 liba2ats_s8; do
  echo "== $v" >> gpurun_out/split.log
  A2ATS_LIB=paper_2502_12665_b200/lib/$v.so timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['roofline']['frac'], d['kernels']['attention']['ms'])" >> gpurun_out/split.log 2>&1
done
