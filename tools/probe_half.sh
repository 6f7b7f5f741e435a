python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_gemm.py -x -q > gpurun_out/pytest_gemm.log 2>&1; echo rc=$? >> gpurun_out/pytest_gemm.log
timeout 900 python -m pytest tests/test_gpu_model.py tests/test_gpu_fullsize.py -x -q > gpurun_out/pytest_model.log 2>&1; echo rc=$? >> gpurun_out/pytest_model.log
SARATHI_MODEL_TRACE=3:320 SARATHI_TRACE_ALL=1 timeout 300 python tools/profile_step.py --steps 1 > gpurun_out/probe_trace_m3_half.txt 2>&1
timeout 300 python tools/profile_step.py --steps 1 --spans 10 > gpurun_out/probe_spans_half.txt 2>&1
bash tools/ab.sh "SARATHI_GEMM_HALF=1" "SARATHI_GEMM_HALF=0"
