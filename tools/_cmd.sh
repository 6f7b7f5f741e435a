python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
SARATHI_PREFILL_BK=128 timeout 300 python tools/shard_step.py > gpurun_out/shard_bk128.log 2>&1
timeout 300 python tools/shard_step.py > gpurun_out/shard_bk64.log 2>&1
