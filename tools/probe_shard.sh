# TP-rank shapes (tools/shard_step.py) with the layer chain on / off
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
SARATHI_CHAIN_PRINT=1 timeout 600 python tools/shard_step.py > gpurun_out/shard_on.txt 2> gpurun_out/shard_on.err
SARATHI_CHAIN=0 timeout 600 python tools/shard_step.py > gpurun_out/shard_off.txt 2> gpurun_out/shard_off.err
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
