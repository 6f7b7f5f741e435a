# compute-sanitizer passes over small GPU schedules: default path, the layer chain (forced, split
# whole tiles) and the flag-gated O projection.  Summaries -> gpurun_out/sanitizer_*.txt
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
SEL="config1 or gelu or block_size_32 or gqa"
for tool in memcheck synccheck racecheck; do
  for cfg in "default:" "chain:SARATHI_CHAIN=2 SARATHI_CHAIN_SPLIT=1" "oearly:SARATHI_O_EARLY=1"; do
    name=${cfg%%:*}; envs=${cfg#*:}
    echo "== $tool $name ($envs)" >> gpurun_out/sanitizer_$tool.txt
    env $envs SARATHI_PREFILL_VARIANT_CHILD=1 timeout 1200 compute-sanitizer --tool $tool --print-limit 20 \
      python -m pytest tests/test_gpu_model.py -q -m gpu -k "$SEL" -p no:cacheprovider 2>&1 | tail -6 >> gpurun_out/sanitizer_$tool.txt
  done
done
