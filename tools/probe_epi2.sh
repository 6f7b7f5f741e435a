# per-chunk epilogue timelines of the standalone QKV (mode 5) and gate||up (mode 3) GEMMs in the model
for m in 5 3 2; do echo "== mode $m"; SARATHI_MODEL_TRACE=$m:320 timeout 200 python tools/profile_step.py --steps 1 2>&1 | grep -E "trace M|seg|CTA end"; done > gpurun_out/epi_probe2.txt 2>&1
