# RMSNorm-as-epilogue of the residual-add GEMMs: model parity tests, a span timeline, A/B vs the
# rmsnorm kernel (SARATHI_POST_NORM=0)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_model.py tests/test_gpu_fullsize.py -x -q > gpurun_out/pytest_model.log 2>&1; echo rc=$? >> gpurun_out/pytest_model.log
timeout 300 python tools/profile_step.py --steps 1 --spans 12 > gpurun_out/probe_spans_pnorm.txt 2>&1
rm -rf gpurun_out/ab
bash tools/ab.sh "SARATHI_POST_NORM=1" "SARATHI_POST_NORM=0"
