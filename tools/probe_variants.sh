# A/B of library variants: var_so/lib*.so swapped in for the bench + chain trace
mkdir -p gpurun_out/var
cp paper_2308_16369_b200/libsarathi.so var_so/libcur.so
for v in var_so/lib*.so; do
  n=$(basename $v .so)
  cp $v paper_2308_16369_b200/libsarathi.so
  SARATHI_CHAIN_PRINT=1 timeout 300 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/var/bench_$n.json 2> gpurun_out/var/bench_$n.err
  SARATHI_CHAIN_TRACE=320 timeout 300 python tools/profile_step.py --steps 5 > gpurun_out/var/trace_$n.txt 2>&1
done
cp var_so/libcur.so paper_2308_16369_b200/libsarathi.so
