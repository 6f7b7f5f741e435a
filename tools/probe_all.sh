# build, GPU tests, GEMM microbench + traces, model bench (timing experiments for the GEMM)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
(SARATHI_GEMM_TRACE=1 timeout 100 python tools/gemm_one.py 15360 320 5120 0; SARATHI_GEMM_TRACE=1 timeout 100 python tools/gemm_one.py 27648 320 5120 3) 2>&1 | grep -E "trace M|seg" > gpurun_out/epi_probe.txt
timeout 200 python tools/gemm_bench.py --n 320 --modes 0 2 3 --iters 5 > gpurun_out/gemm_probe.txt 2>&1
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
