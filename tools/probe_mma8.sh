# Prefill attention S / PV issue as one asm block of 8 UMMAs (SARATHI_ATTN_MMA8, default on):
# model tests, TP-rank shapes and bench A/B
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_model.py tests/test_gpu_fullsize.py -x -q > gpurun_out/pytest_model.log 2>&1; echo rc=$? >> gpurun_out/pytest_model.log
timeout 600 python tools/shard_step.py > gpurun_out/shard_step.txt 2> gpurun_out/shard_step.err
SARATHI_ATTN_MMA8=0 timeout 600 python tools/shard_step.py > gpurun_out/shard_step_m0.txt 2> gpurun_out/shard_step_m0.err
rm -rf gpurun_out/ab
bash tools/ab.sh "SARATHI_ATTN_MMA8=1" "SARATHI_ATTN_MMA8=0"
