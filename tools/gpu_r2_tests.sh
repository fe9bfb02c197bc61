# Round-2: C2 step variants (pipe select at one chunk; qprep for NV = 64)
mkdir -p gpurun_out
for v in liba2ats liba2ats_pipe1 liba2ats_q32 liba2ats_both; do
  echo "== $v" >> gpurun_out/c2_var.log
  A2ATS_LIB=paper_2502_12665_b200/lib/$v.so timeout 600 python bench.py --config C2 --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['scoring']['ms'], d['e2e']['ms_per_step'])" >> gpurun_out/c2_var.log
done
