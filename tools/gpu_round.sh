# Round evidence on one B200: build, GPU tests, bench line, then the ncu launch list and full captures
# (tools/profile_round.sh).  Outputs under gpurun_out/.  EXTRA=1 adds the deterministic-mode and
# layer-chain bench lines.
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
if [ "${EXTRA:-0}" = 1 ]; then
  SARATHI_DETERMINISTIC=1 timeout 300 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/bench_det.json 2>/dev/null
  SARATHI_CHAIN=1 timeout 300 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/bench_chain.json 2>/dev/null
fi
[ "${SKIP_NCU:-0}" = 1 ] || bash tools/profile_round.sh
