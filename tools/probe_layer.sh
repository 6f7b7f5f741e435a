# One layer of the bench composition under the microscope: device-span timeline of one hybrid step
# (PDL chain intact) and the in-kernel timelines of the QKV / O / gate||up GEMMs (pair 0 + every
# pair's end).  Outputs gpurun_out/probe_*.txt.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 300 python tools/profile_step.py --steps 1 --spans 24 > gpurun_out/probe_spans.txt 2>&1
for m in 5 2 3; do
  SARATHI_MODEL_TRACE=$m:320 SARATHI_TRACE_ALL=1 timeout 300 python tools/profile_step.py --steps 1 > gpurun_out/probe_trace_m$m.txt 2>&1
done
