# QKV epilogue components inside the chain (timing only, results invalid): 0 full, 1 no emit,
# 32 no RoPE math, 8 no global stores
mkdir -p gpurun_out/var
cp paper_2308_16369_b200/libsarathi.so var_so/libcur.so
cp var_so/libqkvdbg.so paper_2308_16369_b200/libsarathi.so
for v in 0 1 32 8 40; do
  SARATHI_CHAIN_QKV_DBG=$v SARATHI_CHAIN_TRACE=320 timeout 300 python tools/profile_step.py --steps 5 > gpurun_out/var/qkvdbg_$v.txt 2>&1
done
cp var_so/libcur.so paper_2308_16369_b200/libsarathi.so
