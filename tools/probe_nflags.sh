# Flag-chained RMSNorm (SARATHI_NORM_FLAGS, default on): model tests, span timeline, TP ranks, bench A/B
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_model.py tests/test_gpu_fullsize.py -x -q > gpurun_out/pytest_model.log 2>&1; echo rc=$? >> gpurun_out/pytest_model.log
timeout 300 python tools/profile_step.py --steps 1 --spans 12 > gpurun_out/probe_spans_nf.txt 2>&1
SARATHI_NORM_FLAGS=0 timeout 300 python tools/profile_step.py --steps 1 --spans 12 > gpurun_out/probe_spans_nf0.txt 2>&1
timeout 600 python tools/shard_step.py > gpurun_out/shard_step.txt 2> gpurun_out/shard_step.err
rm -rf gpurun_out/ab
bash tools/ab.sh "SARATHI_NORM_FLAGS=1" "SARATHI_NORM_FLAGS=0"
