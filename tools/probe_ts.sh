# A-from-TMEM GEMM option: exact-integer GEMM tests, per-k-block N sweep, model tests + bench A/B
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
SARATHI_GEMM_TS=1 timeout 600 python -m pytest tests/test_gpu_gemm.py -x -q > gpurun_out/pytest_ts_gemm.log 2>&1; echo rc=$? >> gpurun_out/pytest_ts_gemm.log
for n in 256 272 320 384 448; do
  echo "== N=$n" >> gpurun_out/nsweep_ts.txt
  SARATHI_GEMM_TS=1 SARATHI_GEMM_TRACE=1 timeout 100 python tools/gemm_one.py 15360 $n 5120 0 2>&1 | grep -E "trace M|^u" >> gpurun_out/nsweep_ts.txt
done
SARATHI_GEMM_TS=1 timeout 600 python -m pytest tests/test_gpu_model.py -x -q -k "not variants and not deterministic_mode" > gpurun_out/pytest_ts_model.log 2>&1; echo rc=$? >> gpurun_out/pytest_ts_model.log
mkdir -p gpurun_out/ab4
for r in 1 2; do for t in 1 0; do SARATHI_GEMM_TS=$t timeout 300 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/ab4/ts${t}_r$r.json 2>/dev/null; done; done
