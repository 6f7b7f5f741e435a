# Narrow-token GEMM k-block rate (70B TP-8 rank gate||up M=7168 K=8192 N=282: two token tiles of 144,
# one UMMA per k-step) vs ring stages and vs one 288-token tile; TP-rank shapes baseline
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for st in 8 6 4; do
  echo "== stages $st" >> gpurun_out/narrow.txt
  SARATHI_GEMM_STAGES=$st SARATHI_GEMM_TRACE=1 timeout 100 python tools/gemm_one.py 7168 282 8192 0 2>&1 | grep -E "trace M|^u *(0|1|2|10|20|40|60|80|100|120|127) |CTA end" >> gpurun_out/narrow.txt
done
echo "== one token tile (SARATHI_GEMM_NT_SMALLM=0)" >> gpurun_out/narrow.txt
SARATHI_GEMM_NT_SMALLM=0 SARATHI_GEMM_TRACE=1 timeout 100 python tools/gemm_one.py 7168 282 8192 0 2>&1 | grep -E "trace M|^u *(0|1|2|10|20|40|60|80|100|120|127) |CTA end|seg" >> gpurun_out/narrow.txt
echo "== 13B gate||up T=256 (one UMMA N=256)" >> gpurun_out/narrow.txt
SARATHI_GEMM_TRACE=1 timeout 100 python tools/gemm_one.py 27648 256 5120 0 2>&1 | grep -E "trace M|^u *(0|1|2|10|20|40|60|79|80|100|115) |CTA end|seg" >> gpurun_out/narrow.txt
echo "== 13B gate||up T=320" >> gpurun_out/narrow.txt
SARATHI_GEMM_TRACE=1 timeout 100 python tools/gemm_one.py 27648 320 5120 0 2>&1 | grep -E "trace M|^u *(0|1|2|10|20|40|60|79|80|100|115) |CTA end|seg" >> gpurun_out/narrow.txt
timeout 600 python tools/shard_step.py > gpurun_out/shard_step.txt 2> gpurun_out/shard_step.err
