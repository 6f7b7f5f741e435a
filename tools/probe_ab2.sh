# interleaved A/B of library variants (two rounds), hybrid bench only; then the GPU tests on the default
mkdir -p gpurun_out/ab2
cp paper_2308_16369_b200/libsarathi.so var_so/libkeep.so
for r in 1 2; do
  for v in ${VARIANTS:-libcur libD}; do
    cp var_so/$v.so paper_2308_16369_b200/libsarathi.so
    timeout 300 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/ab2/${v}_r$r.json 2>/dev/null
  done
done
cp var_so/libkeep.so paper_2308_16369_b200/libsarathi.so
[ "${FULL:-0}" = 1 ] && { timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log; }
true
