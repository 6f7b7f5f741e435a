python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for d in 0 1 2 3; do echo "== DBG=$d"; SARATHI_GEMM_DBG=$d timeout 200 python tools/gemm_bench.py --n 320 --modes 0 2 --iters 5; done > gpurun_out/gemm_probe4.txt 2>&1
for st in 3 4; do echo "== STAGES=$st"; SARATHI_GEMM_STAGES=$st timeout 200 python tools/gemm_bench.py --n 320 --modes 0 2 --iters 5; done >> gpurun_out/gemm_probe4.txt 2>&1
(SARATHI_GEMM_TRACE=1 timeout 100 python tools/gemm_one.py 15360 320 5120 0; SARATHI_GEMM_TRACE=1 timeout 100 python tools/gemm_one.py 27648 320 5120 3; SARATHI_GEMM_TRACE=1 timeout 100 python tools/gemm_one.py 5120 320 5120 2) > gpurun_out/gemm_trace3.txt 2>&1
