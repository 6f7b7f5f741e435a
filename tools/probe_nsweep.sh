# per-k-block MMA time of one GEMM (M=15360, K=5120, store epilogue) vs token count N
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for n in 128 192 256 272 288 320 352 384 448 512; do
  echo "== N=$n" >> gpurun_out/nsweep.txt
  SARATHI_GEMM_TRACE=1 timeout 100 python tools/gemm_one.py 15360 $n 5120 0 2>&1 | grep -E "trace M|^u" >> gpurun_out/nsweep.txt
  SARATHI_GEMM_UNEVEN=0 SARATHI_GEMM_TRACE=1 timeout 100 python tools/gemm_one.py 15360 $n 5120 0 2>&1 | grep -E "trace M" | sed 's/^/even: /' >> gpurun_out/nsweep.txt
done
