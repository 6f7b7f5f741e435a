python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for d in 0 4 8; do echo "== DBG=$d"; (SARATHI_GEMM_DBG=$d SARATHI_GEMM_TRACE=1 timeout 100 python tools/gemm_one.py 15360 320 5120 0; SARATHI_GEMM_DBG=$d SARATHI_GEMM_TRACE=1 timeout 100 python tools/gemm_one.py 27648 320 5120 3) 2>&1 | grep -E "trace M|seg"; done > gpurun_out/epi_probe.txt 2>&1
timeout 200 python tools/gemm_bench.py --n 320 --modes 0 2 3 --iters 5 > gpurun_out/gemm_probe5.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_gemm.py -x -q > gpurun_out/pytest_gemm.log 2>&1
