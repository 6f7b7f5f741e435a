# T = 256 (one UMMA per k-step) with / without the one-asm k-block issue, interleaved
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for r in 1 2; do for kb in 1 0; do
  echo "== r$r kbasm=$kb" >> gpurun_out/t256.txt
  SARATHI_GEMM_KBASM=$kb timeout 300 python tools/cliff.py --cases 256:0 256:1 256:64 >> gpurun_out/t256.txt 2>/dev/null
done; done
