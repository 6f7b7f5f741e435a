# Interleaved A/B of environment settings on one box (the box's power-capped clock moves a single
# bench line by +-1 %, so variants alternate and repeat):
#   bash tools/ab.sh "SARATHI_GEMM_TS=1" "SARATHI_GEMM_TS=0"        -> gpurun_out/ab/<i>_r<r>.json
# Used for every kept-or-dropped decision in DESIGN.md §6 (profiles/r02_ab_*.txt).
mkdir -p gpurun_out/ab
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for r in 1 2; do
  i=0
  for v in "$@"; do
    env $v timeout 300 python bench.py --no-cpu-baseline --steps ${STEPS:-20} > gpurun_out/ab/${i}_r$r.json 2>/dev/null
    echo "$i: $v" > gpurun_out/ab/${i}.env
    i=$((i + 1))
  done
done
