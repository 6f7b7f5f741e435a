# Round evidence on one B200: build, GPU tests, bench line, then the ncu launch list and full captures
# (tools/profile_round.sh).  Outputs under gpurun_out/.
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
[ "${SKIP_NCU:-0}" = 1 ] || bash tools/profile_round.sh
