# early O projection (per-head flags) : GPU tests, then interleaved A/B vs SARATHI_O_EARLY=0
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
mkdir -p gpurun_out/ab3
for r in 1 2; do
  for e in 1 0; do
    SARATHI_O_EARLY=$e timeout 300 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/ab3/oearly${e}_r$r.json 2>/dev/null
  done
done
SARATHI_SPANS_ONLY=1 SARATHI_SPAN_DUMP=30 timeout 300 python bench.py --no-cpu-baseline --steps 3 > /dev/null 2> gpurun_out/spans_oearly.txt
