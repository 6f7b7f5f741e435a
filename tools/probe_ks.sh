# prefill-only steps (T = 256): prefill-attention key split forced 2 / 3 vs the cost model
for r in 1 2; do for k in 0 2 3; do
  if [ $k = 0 ]; then timeout 300 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/ks/ks${k}_r$r.json 2>/dev/null;
  else SARATHI_PREFILL_KSPLIT=$k timeout 300 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/ks/ks${k}_r$r.json 2>/dev/null; fi
done; done
