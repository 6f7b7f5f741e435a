# final round evidence: build, all GPU tests, bench line (+ deterministic line), TP-rank shapes, the
# 256-token boundary and the decode sweep at P = 1024, ncu launch list + full captures
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
SARATHI_DETERMINISTIC=1 timeout 300 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/bench_det.json 2>/dev/null
timeout 600 python tools/shard_step.py > gpurun_out/shard_step.txt 2> gpurun_out/shard_step.err
timeout 300 python tools/cliff.py > gpurun_out/cliff.txt 2> gpurun_out/cliff.err
timeout 600 python tools/decode_sweep.py --prompts 1024 > gpurun_out/decode_sweep.txt 2> gpurun_out/decode_sweep.err
bash tools/profile_round.sh
