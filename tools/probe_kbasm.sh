# One-asm-block k-block MMA issue (SARATHI_GEMM_KBASM, default on): GEMM tests, k-block rates
# (no loads / real) at N = 144 / 256 / 320, TP-rank shapes, bench A/B
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_gemm.py -x -q > gpurun_out/pytest_gemm.log 2>&1; echo rc=$? >> gpurun_out/pytest_gemm.log
run() { echo "== $1" >> gpurun_out/kbasm.txt; shift; env "$@" SARATHI_GEMM_TRACE=1 timeout 100 python tools/gemm_one.py $GEMM 2>&1 | grep -E "trace M|^u *(10|60|110) |CTA end" | tail -n 4 >> gpurun_out/kbasm.txt; }
for kb in 1 0; do
GEMM="7168 282 8192 0"; run "kbasm=$kb 70B gate_up N=282 (bn 144)" SARATHI_GEMM_KBASM=$kb
GEMM="7168 282 8192 0"; run "kbasm=$kb N=282 skip both" SARATHI_GEMM_KBASM=$kb SARATHI_GEMM_DBG=3
GEMM="27648 256 5120 0"; run "kbasm=$kb 13B gate_up T=256" SARATHI_GEMM_KBASM=$kb
GEMM="27648 256 5120 0"; run "kbasm=$kb T=256 skip both" SARATHI_GEMM_KBASM=$kb SARATHI_GEMM_DBG=3
GEMM="27648 320 5120 0"; run "kbasm=$kb T=320" SARATHI_GEMM_KBASM=$kb
GEMM="27648 320 5120 0"; run "kbasm=$kb T=320 skip both" SARATHI_GEMM_KBASM=$kb SARATHI_GEMM_DBG=3
done
timeout 900 python -m pytest tests/test_gpu_model.py tests/test_gpu_fullsize.py -x -q > gpurun_out/pytest_model.log 2>&1; echo rc=$? >> gpurun_out/pytest_model.log
timeout 600 python tools/shard_step.py > gpurun_out/shard_step.txt 2> gpurun_out/shard_step.err
SARATHI_GEMM_KBASM=0 timeout 600 python tools/shard_step.py > gpurun_out/shard_step_kb0.txt 2> gpurun_out/shard_step_kb0.err
rm -rf gpurun_out/ab
bash tools/ab.sh "SARATHI_GEMM_KBASM=1" "SARATHI_GEMM_KBASM=0"
