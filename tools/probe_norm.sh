# fused RMSNorm prologue: GPU tests, then interleaved A/B vs SARATHI_NORM_FUSED=0
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_model.py tests/test_gpu_fullsize.py -x -q -k "not variants and not chain and not deterministic_mode" > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
mkdir -p gpurun_out/ab5
for r in 1 2; do for e in 1 0; do SARATHI_NORM_FUSED=$e timeout 300 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/ab5/norm${e}_r$r.json 2>/dev/null; done; done
SARATHI_SPANS_ONLY=1 SARATHI_SPAN_DUMP=24 timeout 300 python bench.py --no-cpu-baseline --steps 3 > /dev/null 2> gpurun_out/spans_norm.txt
