# chain kernel: timing + one traced launch (layer 1 of the bench composition)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_model.py -x -q > gpurun_out/pytest_model.log 2>&1; echo rc=$? >> gpurun_out/pytest_model.log
SARATHI_CHAIN_PRINT=1 timeout 300 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench_chain.json 2> gpurun_out/bench_chain.err
SARATHI_CHAIN_TRACE=320 timeout 300 python tools/profile_step.py --steps 1 > gpurun_out/chain_trace.txt 2>&1
