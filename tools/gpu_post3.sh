mkdir -p gpurun_out
L=paper_2502_12665_b200/lib
for v in liba2ats liba2ats_s2 liba2ats_s3; do
  A2ATS_LIB=$L/$v.so timeout 300 python tools/kbench.py --config C2 --no-append --iters 8 > gpurun_out/kb_c2_$v.log 2>&1
done
timeout 600 python bench.py --config C2 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
