# TMEM-slot releases by relaxed cluster arrives (SARATHI_GEMM_RELAXED, default on) vs release.cluster
# (MEMBAR.ALL.GPU per arrive): GEMM + model tests, in-model traces, TP ranks, bench A/B
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_gemm.py -x -q > gpurun_out/pytest_gemm.log 2>&1; echo rc=$? >> gpurun_out/pytest_gemm.log
timeout 900 python -m pytest tests/test_gpu_model.py tests/test_gpu_fullsize.py -x -q > gpurun_out/pytest_model.log 2>&1; echo rc=$? >> gpurun_out/pytest_model.log
for m in 5 3; do
  SARATHI_MODEL_TRACE=$m:320 timeout 300 python tools/profile_step.py --steps 1 > gpurun_out/rtrace_m$m.txt 2>&1
  SARATHI_GEMM_RELAXED=0 SARATHI_MODEL_TRACE=$m:320 timeout 300 python tools/profile_step.py --steps 1 > gpurun_out/rtrace0_m$m.txt 2>&1
done
timeout 600 python tools/shard_step.py > gpurun_out/shard_step.txt 2> gpurun_out/shard_step.err
SARATHI_GEMM_RELAXED=0 timeout 600 python tools/shard_step.py > gpurun_out/shard_step_r0.txt 2> gpurun_out/shard_step_r0.err
rm -rf gpurun_out/ab
bash tools/ab.sh "SARATHI_GEMM_RELAXED=1" "SARATHI_GEMM_RELAXED=0"
