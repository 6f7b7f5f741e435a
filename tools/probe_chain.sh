# chain kernel: GPU tests, timing + one traced launch (a warm in-model launch of the bench composition)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_model.py -x -q > gpurun_out/pytest_model.log 2>&1; echo rc=$? >> gpurun_out/pytest_model.log
SARATHI_CHAIN_PRINT=1 timeout 300 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench_chain.json 2> gpurun_out/bench_chain.err
SARATHI_CHAIN_TRACE=320 timeout 300 python tools/profile_step.py --steps 5 > gpurun_out/chain_trace.txt 2>&1
[ "${SHARD:-0}" = 1 ] && { SARATHI_CHAIN_PRINT=1 timeout 600 python tools/shard_step.py > gpurun_out/shard_on.txt 2> gpurun_out/shard_on.err; }
[ "${FULL:-0}" = 1 ] && { timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log; }
true
