python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
mkdir -p gpurun_out/shard
for v in "X=0" "SARATHI_GEMM_NT_SMALLM=0" "SARATHI_GEMM_NT_SMALLM=3" "SARATHI_GEMM_NT_SMALLM=4" "SARATHI_GEMM_SK_COST=0.25" "SARATHI_GEMM_SK_COST=1.0" "SARATHI_GEMM_TS=0"; do
  env $v timeout 600 python tools/shard_step.py --which llama70b-tp8 gpt3-tp8 > gpurun_out/shard/$(echo $v | tr '=' '_').txt 2>/dev/null
done
