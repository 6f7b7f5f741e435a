# ncu evidence for profiles/: launch list of bench.py's timed hybrid steps + full captures of the
# decode attention, prefill attention and the four layer GEMMs (one layer) of the bench composition.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
SARATHI_PROFILE_TIMED=1 timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
  --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k "regex:decode_attn" -c 1 \
  -o gpurun_out/prof_decode python tools/profile_step.py --steps 1 > gpurun_out/ncu_decode.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k "regex:gemm|prefill" -c 5 \
  -o gpurun_out/prof_gemm python tools/profile_step.py --steps 1 > gpurun_out/ncu_gemm.log 2>&1
