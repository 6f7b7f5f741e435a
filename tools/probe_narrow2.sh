# What bounds the k-block rate of narrow-token GEMMs: pair count (aggregate bandwidth) or per-pair
# latency; X-only / W-only loads (SARATHI_GEMM_DBG bits 0/1, results invalid)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
run() { echo "== $1" >> gpurun_out/narrow2.txt; shift; env "$@" SARATHI_GEMM_TRACE=1 timeout 100 python tools/gemm_one.py $GEMM 2>&1 | grep -E "trace M|^u *(10|60|110) |CTA end" | tail -n 4 >> gpurun_out/narrow2.txt; }
GEMM="7168 282 8192 0"; run "70B gate_up N=282 (56 pairs, bn 144)" X=1
GEMM="7168 141 8192 0"; run "N=141 (28 pairs)" X=1
GEMM="3584 282 8192 0"; run "M=3584 N=282 (28 pairs, bn 144)" X=1
GEMM="7168 282 8192 0"; run "N=282 skip X loads" SARATHI_GEMM_DBG=1
GEMM="7168 282 8192 0"; run "N=282 skip W loads" SARATHI_GEMM_DBG=2
GEMM="7168 282 8192 0"; run "N=282 skip both" SARATHI_GEMM_DBG=3
GEMM="27648 256 5120 0"; run "13B gate_up T=256 (74 pairs)" X=1
GEMM="27648 256 5120 0"; run "T=256 skip X" SARATHI_GEMM_DBG=1
GEMM="27648 256 5120 0"; run "T=256 skip W" SARATHI_GEMM_DBG=2
GEMM="27648 256 5120 0"; run "T=256 skip both" SARATHI_GEMM_DBG=3
GEMM="27648 320 5120 0"; run "T=320 (74 pairs)" X=1
GEMM="27648 320 5120 0"; run "T=320 skip both" SARATHI_GEMM_DBG=3
