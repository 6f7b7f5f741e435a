# chain on/off A/B in one box (alternating, 2 runs each) + one device-span timeline of a hybrid step
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for i in 1 2; do
  SARATHI_CHAIN=0 timeout 300 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/ab_off_$i.json 2>/dev/null
  SARATHI_CHAIN=1 timeout 300 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/ab_on_$i.json 2>/dev/null
done
SARATHI_SPANS_ONLY=1 SARATHI_SPAN_DUMP=40 timeout 300 python bench.py --no-cpu-baseline --steps 3 > /dev/null 2> gpurun_out/spans_on.txt
SARATHI_CHAIN=0 SARATHI_SPANS_ONLY=1 SARATHI_SPAN_DUMP=40 timeout 300 python bench.py --no-cpu-baseline --steps 3 > /dev/null 2> gpurun_out/spans_off.txt
