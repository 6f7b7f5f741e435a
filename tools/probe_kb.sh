# per-k-block MMA timelines of the layer GEMMs at T=320 (hybrid) and T=256 (prefill-only)
for spec in 5:320 2:320 3:320 5:256; do
  kind=hybrid; [ "${spec#*:}" = 256 ] && kind=prefill
  SARATHI_MODEL_TRACE=$spec timeout 200 python tools/profile_step.py --steps 1 --kind $kind 2>&1 | grep -E "trace M|^u" > gpurun_out/kb_${spec/:/_}.txt
done
SARATHI_GEMM_UNEVEN=0 SARATHI_MODEL_TRACE=5:320 timeout 200 python tools/profile_step.py --steps 1 2>&1 | grep -E "trace M|^u" > gpurun_out/kb_5_320_even.txt
