#!/bin/bash
# Every GPU experiment behind a DESIGN.md §6 number, one case per experiment (run under gpurun;
# outputs under gpurun_out/).  Usage: bash tools/experiments.sh <name> [<name> ...]
#   half kbasm layer mma8 narrow narrow2 nflags nsweep pnorm relaxed t256 ts
build() { python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; }
mkdir -p gpurun_out
for exp in "$@"; do
case "$exp" in
half)
  build
  timeout 600 python -m pytest tests/test_gpu_gemm.py -x -q > gpurun_out/pytest_gemm.log 2>&1; echo rc=$? >> gpurun_out/pytest_gemm.log
  timeout 900 python -m pytest tests/test_gpu_model.py tests/test_gpu_fullsize.py -x -q > gpurun_out/pytest_model.log 2>&1; echo rc=$? >> gpurun_out/pytest_model.log
  SARATHI_MODEL_TRACE=3:320 SARATHI_TRACE_ALL=1 timeout 300 python tools/profile_step.py --steps 1 > gpurun_out/probe_trace_m3_half.txt 2>&1
  timeout 300 python tools/profile_step.py --steps 1 --spans 10 > gpurun_out/probe_spans_half.txt 2>&1
  bash tools/ab.sh "SARATHI_GEMM_HALF=1" "SARATHI_GEMM_HALF=0"
  ;;
kbasm)
  # One-asm-block k-block MMA issue (SARATHI_GEMM_KBASM, default on): GEMM tests, k-block rates
  # (no loads / real) at N = 144 / 256 / 320, TP-rank shapes, bench A/B
  build
  timeout 600 python -m pytest tests/test_gpu_gemm.py -x -q > gpurun_out/pytest_gemm.log 2>&1; echo rc=$? >> gpurun_out/pytest_gemm.log
  run() { echo "== $1" >> gpurun_out/kbasm.txt; shift; env "$@" SARATHI_GEMM_TRACE=1 timeout 100 python tools/gemm_one.py $GEMM 2>&1 | grep -E "trace M|^u *(10|60|110) |CTA end" | tail -n 4 >> gpurun_out/kbasm.txt; }
  for kb in 1 0; do
  GEMM="7168 282 8192 0"; run "kbasm=$kb 70B gate_up N=282 (bn 144)" SARATHI_GEMM_KBASM=$kb
  GEMM="7168 282 8192 0"; run "kbasm=$kb N=282 skip both" SARATHI_GEMM_KBASM=$kb SARATHI_GEMM_DBG=3
  GEMM="27648 256 5120 0"; run "kbasm=$kb 13B gate_up T=256" SARATHI_GEMM_KBASM=$kb
  GEMM="27648 256 5120 0"; run "kbasm=$kb T=256 skip both" SARATHI_GEMM_KBASM=$kb SARATHI_GEMM_DBG=3
  GEMM="27648 320 5120 0"; run "kbasm=$kb T=320" SARATHI_GEMM_KBASM=$kb
  GEMM="27648 320 5120 0"; run "kbasm=$kb T=320 skip both" SARATHI_GEMM_KBASM=$kb SARATHI_GEMM_DBG=3
  done
  timeout 900 python -m pytest tests/test_gpu_model.py tests/test_gpu_fullsize.py -x -q > gpurun_out/pytest_model.log 2>&1; echo rc=$? >> gpurun_out/pytest_model.log
  timeout 600 python tools/shard_step.py > gpurun_out/shard_step.txt 2> gpurun_out/shard_step.err
  SARATHI_GEMM_KBASM=0 timeout 600 python tools/shard_step.py > gpurun_out/shard_step_kb0.txt 2> gpurun_out/shard_step_kb0.err
  rm -rf gpurun_out/ab
  bash tools/ab.sh "SARATHI_GEMM_KBASM=1" "SARATHI_GEMM_KBASM=0"
  ;;
layer)
  # One layer of the bench composition under the microscope: device-span timeline of one hybrid step
  # (PDL chain intact) and the in-kernel timelines of the QKV / O / gate||up GEMMs (pair 0 + every
  # pair's end).  Outputs gpurun_out/probe_*.txt.
  build
  timeout 300 python tools/profile_step.py --steps 1 --spans 24 > gpurun_out/probe_spans.txt 2>&1
  for m in 5 2 3; do
    SARATHI_MODEL_TRACE=$m:320 SARATHI_TRACE_ALL=1 timeout 300 python tools/profile_step.py --steps 1 > gpurun_out/probe_trace_m$m.txt 2>&1
  done
  ;;
mma8)
  # Prefill attention S / PV issue as one asm block of 8 UMMAs (SARATHI_ATTN_MMA8, default on):
  # model tests, TP-rank shapes and bench A/B
  build
  timeout 900 python -m pytest tests/test_gpu_model.py tests/test_gpu_fullsize.py -x -q > gpurun_out/pytest_model.log 2>&1; echo rc=$? >> gpurun_out/pytest_model.log
  timeout 600 python tools/shard_step.py > gpurun_out/shard_step.txt 2> gpurun_out/shard_step.err
  SARATHI_ATTN_MMA8=0 timeout 600 python tools/shard_step.py > gpurun_out/shard_step_m0.txt 2> gpurun_out/shard_step_m0.err
  rm -rf gpurun_out/ab
  bash tools/ab.sh "SARATHI_ATTN_MMA8=1" "SARATHI_ATTN_MMA8=0"
  ;;
narrow)
  # Narrow-token GEMM k-block rate (70B TP-8 rank gate||up M=7168 K=8192 N=282: two token tiles of 144,
  # one UMMA per k-step) vs ring stages and vs one 288-token tile; TP-rank shapes baseline
  build
  for st in 8 6 4; do
    echo "== stages $st" >> gpurun_out/narrow.txt
    SARATHI_GEMM_STAGES=$st SARATHI_GEMM_TRACE=1 timeout 100 python tools/gemm_one.py 7168 282 8192 0 2>&1 | grep -E "trace M|^u *(0|1|2|10|20|40|60|80|100|120|127) |CTA end" >> gpurun_out/narrow.txt
  done
  echo "== one token tile (SARATHI_GEMM_NT_SMALLM=0)" >> gpurun_out/narrow.txt
  SARATHI_GEMM_NT_SMALLM=0 SARATHI_GEMM_TRACE=1 timeout 100 python tools/gemm_one.py 7168 282 8192 0 2>&1 | grep -E "trace M|^u *(0|1|2|10|20|40|60|80|100|120|127) |CTA end|seg" >> gpurun_out/narrow.txt
  echo "== 13B gate||up T=256 (one UMMA N=256)" >> gpurun_out/narrow.txt
  SARATHI_GEMM_TRACE=1 timeout 100 python tools/gemm_one.py 27648 256 5120 0 2>&1 | grep -E "trace M|^u *(0|1|2|10|20|40|60|79|80|100|115) |CTA end|seg" >> gpurun_out/narrow.txt
  echo "== 13B gate||up T=320" >> gpurun_out/narrow.txt
  SARATHI_GEMM_TRACE=1 timeout 100 python tools/gemm_one.py 27648 320 5120 0 2>&1 | grep -E "trace M|^u *(0|1|2|10|20|40|60|79|80|100|115) |CTA end|seg" >> gpurun_out/narrow.txt
  timeout 600 python tools/shard_step.py > gpurun_out/shard_step.txt 2> gpurun_out/shard_step.err
  ;;
narrow2)
  # What bounds the k-block rate of narrow-token GEMMs: pair count (aggregate bandwidth) or per-pair
  # latency; X-only / W-only loads (SARATHI_GEMM_DBG bits 0/1, results invalid)
  build
  run() { echo "== $1" >> gpurun_out/narrow2.txt; shift; env "$@" SARATHI_GEMM_TRACE=1 timeout 100 python tools/gemm_one.py $GEMM 2>&1 | grep -E "trace M|^u *(10|60|110) |CTA end" | tail -n 4 >> gpurun_out/narrow2.txt; }
  GEMM="7168 282 8192 0"; run "70B gate_up N=282 (56 pairs, bn 144)" X=1
  GEMM="7168 141 8192 0"; run "N=141 (28 pairs)" X=1
  GEMM="3584 282 8192 0"; run "M=3584 N=282 (28 pairs, bn 144)" X=1
  GEMM="7168 282 8192 0"; run "N=282 skip X loads" SARATHI_GEMM_DBG=1
  GEMM="7168 282 8192 0"; run "N=282 skip W loads" SARATHI_GEMM_DBG=2
  GEMM="7168 282 8192 0"; run "N=282 skip both" SARATHI_GEMM_DBG=3
  GEMM="27648 256 5120 0"; run "13B gate_up T=256 (74 pairs)" X=1
  GEMM="27648 256 5120 0"; run "T=256 skip X" SARATHI_GEMM_DBG=1
  GEMM="27648 256 5120 0"; run "T=256 skip W" SARATHI_GEMM_DBG=2
  GEMM="27648 256 5120 0"; run "T=256 skip both" SARATHI_GEMM_DBG=3
  GEMM="27648 320 5120 0"; run "T=320 (74 pairs)" X=1
  GEMM="27648 320 5120 0"; run "T=320 skip both" SARATHI_GEMM_DBG=3
  ;;
nflags)
  # Flag-chained RMSNorm (SARATHI_NORM_FLAGS, default on): model tests, span timeline, TP ranks, bench A/B
  build
  timeout 900 python -m pytest tests/test_gpu_model.py tests/test_gpu_fullsize.py -x -q > gpurun_out/pytest_model.log 2>&1; echo rc=$? >> gpurun_out/pytest_model.log
  timeout 300 python tools/profile_step.py --steps 1 --spans 12 > gpurun_out/probe_spans_nf.txt 2>&1
  SARATHI_NORM_FLAGS=0 timeout 300 python tools/profile_step.py --steps 1 --spans 12 > gpurun_out/probe_spans_nf0.txt 2>&1
  timeout 600 python tools/shard_step.py > gpurun_out/shard_step.txt 2> gpurun_out/shard_step.err
  rm -rf gpurun_out/ab
  bash tools/ab.sh "SARATHI_NORM_FLAGS=1" "SARATHI_NORM_FLAGS=0"
  ;;
nsweep)
  # per-k-block MMA time of one GEMM (M=15360, K=5120, store epilogue) vs token count N
  build
  for n in 128 192 256 272 288 320 352 384 448 512; do
    echo "== N=$n" >> gpurun_out/nsweep.txt
    SARATHI_GEMM_TRACE=1 timeout 100 python tools/gemm_one.py 15360 $n 5120 0 2>&1 | grep -E "trace M|^u" >> gpurun_out/nsweep.txt
    SARATHI_GEMM_UNEVEN=0 SARATHI_GEMM_TRACE=1 timeout 100 python tools/gemm_one.py 15360 $n 5120 0 2>&1 | grep -E "trace M" | sed 's/^/even: /' >> gpurun_out/nsweep.txt
  done
  ;;
pnorm)
  # RMSNorm-as-epilogue of the residual-add GEMMs: model parity tests, a span timeline, A/B vs the
  # rmsnorm kernel (SARATHI_POST_NORM=0)
  build
  timeout 900 python -m pytest tests/test_gpu_model.py tests/test_gpu_fullsize.py -x -q > gpurun_out/pytest_model.log 2>&1; echo rc=$? >> gpurun_out/pytest_model.log
  timeout 300 python tools/profile_step.py --steps 1 --spans 12 > gpurun_out/probe_spans_pnorm.txt 2>&1
  rm -rf gpurun_out/ab
  bash tools/ab.sh "SARATHI_POST_NORM=1" "SARATHI_POST_NORM=0"
  ;;
relaxed)
  # TMEM-slot releases by relaxed cluster arrives (SARATHI_GEMM_RELAXED, default on) vs release.cluster
  # (MEMBAR.ALL.GPU per arrive): GEMM + model tests, in-model traces, TP ranks, bench A/B
  build
  timeout 600 python -m pytest tests/test_gpu_gemm.py -x -q > gpurun_out/pytest_gemm.log 2>&1; echo rc=$? >> gpurun_out/pytest_gemm.log
  timeout 900 python -m pytest tests/test_gpu_model.py tests/test_gpu_fullsize.py -x -q > gpurun_out/pytest_model.log 2>&1; echo rc=$? >> gpurun_out/pytest_model.log
  for m in 5 3; do
    SARATHI_MODEL_TRACE=$m:320 timeout 300 python tools/profile_step.py --steps 1 > gpurun_out/rtrace_m$m.txt 2>&1
    SARATHI_GEMM_RELAXED=0 SARATHI_MODEL_TRACE=$m:320 timeout 300 python tools/profile_step.py --steps 1 > gpurun_out/rtrace0_m$m.txt 2>&1
  done
  timeout 600 python tools/shard_step.py > gpurun_out/shard_step.txt 2> gpurun_out/shard_step.err
  SARATHI_GEMM_RELAXED=0 timeout 600 python tools/shard_step.py > gpurun_out/shard_step_r0.txt 2> gpurun_out/shard_step_r0.err
  rm -rf gpurun_out/ab
  bash tools/ab.sh "SARATHI_GEMM_RELAXED=1" "SARATHI_GEMM_RELAXED=0"
  ;;
t256)
  # T = 256 (one UMMA per k-step) with / without the one-asm k-block issue, interleaved
  build
  for r in 1 2; do for kb in 1 0; do
    echo "== r$r kbasm=$kb" >> gpurun_out/t256.txt
    SARATHI_GEMM_KBASM=$kb timeout 300 python tools/cliff.py --cases 256:0 256:1 256:64 >> gpurun_out/t256.txt 2>/dev/null
  done; done
  ;;
ts)
  # A-from-TMEM GEMM option: exact-integer GEMM tests, per-k-block N sweep, model tests + bench A/B
  build
  SARATHI_GEMM_TS=1 timeout 600 python -m pytest tests/test_gpu_gemm.py -x -q > gpurun_out/pytest_ts_gemm.log 2>&1; echo rc=$? >> gpurun_out/pytest_ts_gemm.log
  for n in 256 272 320 384 448; do
    echo "== N=$n" >> gpurun_out/nsweep_ts.txt
    SARATHI_GEMM_TS=1 SARATHI_GEMM_TRACE=1 timeout 100 python tools/gemm_one.py 15360 $n 5120 0 2>&1 | grep -E "trace M|^u" >> gpurun_out/nsweep_ts.txt
  done
  SARATHI_GEMM_TS=1 timeout 600 python -m pytest tests/test_gpu_model.py -x -q -k "not variants and not deterministic_mode" > gpurun_out/pytest_ts_model.log 2>&1; echo rc=$? >> gpurun_out/pytest_ts_model.log
  mkdir -p gpurun_out/ab4
  for r in 1 2; do for t in 1 0; do SARATHI_GEMM_TS=$t timeout 300 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/ab4/ts${t}_r$r.json 2>/dev/null; done; done
  ;;
ntsmall)
  # TP-rank shapes with / without the small-M token split (SARATHI_GEMM_NT_SMALLM=0), after the MMA-issue fix
  build
  for r in 1 2; do for v in 2 0; do
    echo "== r$r nt_smallm=$v" >> gpurun_out/ntsmall.txt
    SARATHI_GEMM_NT_SMALLM=$v timeout 600 python tools/shard_step.py >> gpurun_out/ntsmall.txt 2>/dev/null
  done; done
  ;;
sweep)
  # chunk / tile sweep (NEXT-2) and the zipf request workload on the session-3 kernels
  build
  timeout 1500 python tools/chunk_sweep.py --reps 2 > gpurun_out/chunk_sweep.txt 2> gpurun_out/chunk_sweep.err
  timeout 900 python bench.py --workload zipf-p10-llama13b --no-cpu-baseline > gpurun_out/bench_zipf.json 2> gpurun_out/bench_zipf.err
  ;;
epi)
  # in-model QKV epilogue components (pair 0 trace): full, TMEM loads only (dbg 4), no RoPE (32),
  # no global stores (8); plus the issue-variant GEMM tests
  build
  for dbg in 0 4 32 8; do
    echo "== dbg $dbg" >> gpurun_out/epi_model.txt
    SARATHI_GEMM_DBG=$dbg SARATHI_MODEL_TRACE=5:320 timeout 300 python tools/profile_step.py --steps 1 2>&1 | grep -E "CTA end|seg|chunk" >> gpurun_out/epi_model.txt
  done
  timeout 900 python -m pytest tests/test_gpu_gemm.py -x -q -k "variants" > gpurun_out/pytest_gemm_var.log 2>&1; echo rc=$? >> gpurun_out/pytest_gemm_var.log
  ;;
ropetab)
  # per-batch RoPE (cos, sin) table read by the QKV epilogue (SARATHI_ROPE_TABLE, default on)
  build
  timeout 900 python -m pytest tests/test_gpu_model.py tests/test_gpu_fullsize.py tests/test_gpu_tp_local.py -x -q > gpurun_out/pytest_model.log 2>&1; echo rc=$? >> gpurun_out/pytest_model.log
  for v in 1 0; do
    echo "== rope_table=$v" >> gpurun_out/ropetab.txt
    SARATHI_ROPE_TABLE=$v SARATHI_MODEL_TRACE=5:320 timeout 300 python tools/profile_step.py --steps 1 2>&1 | grep -E "CTA end|seg|chunk (0|2|10|16|18) " >> gpurun_out/ropetab.txt
  done
  timeout 600 python tools/shard_step.py > gpurun_out/shard_step.txt 2> gpurun_out/shard_step.err
  rm -rf gpurun_out/ab
  bash tools/ab.sh "SARATHI_ROPE_TABLE=1" "SARATHI_ROPE_TABLE=0"
  ;;
chainkb)
  # the layer chain with the one-asm k-block issue + relaxed slot releases vs the standalone GEMMs
  build
  timeout 1500 python -m pytest tests/test_gpu_model.py -x -q -k "chain" > gpurun_out/pytest_chain.log 2>&1; echo rc=$? >> gpurun_out/pytest_chain.log
  rm -rf gpurun_out/ab
  bash tools/ab.sh "SARATHI_CHAIN=1" "SARATHI_CHAIN=0"
  SARATHI_CHAIN=1 timeout 600 python tools/shard_step.py > gpurun_out/shard_step_chain.txt 2>/dev/null
  ;;
ppb)
  # pipeline bubbles (paper §5.3, NEXT-4) with stage costs measured on the session-3 kernels
  build
  timeout 1200 python tools/pp_bubbles.py > gpurun_out/pp_bubbles.txt 2> gpurun_out/pp_bubbles.err
  ;;
pairbar)
  # prefill attention: row-half max exchange through per-quarter 2-warp barriers (SARATHI_PREFILL_PAIRBAR)
  build
  timeout 900 python -m pytest tests/test_gpu_model.py tests/test_gpu_fullsize.py -x -q > gpurun_out/pytest_model.log 2>&1; echo rc=$? >> gpurun_out/pytest_model.log
  for v in 1 0; do
    echo "== pairbar=$v" >> gpurun_out/pairbar.txt
    SARATHI_PREFILL_PAIRBAR=$v timeout 600 python tools/shard_step.py >> gpurun_out/pairbar.txt 2>/dev/null
    SARATHI_PREFILL_PAIRBAR=$v timeout 300 python tools/cliff.py --cases 256:0 >> gpurun_out/pairbar.txt 2>/dev/null
  done
  rm -rf gpurun_out/ab
  bash tools/ab.sh "SARATHI_PREFILL_PAIRBAR=1" "SARATHI_PREFILL_PAIRBAR=0"
  ;;
pdsweep)
  # paper §5.2 Fig. orca: (b) P:D sweep at 1K (chunks 256 / 512 vs Orca best / request-level);
  # (a) the balanced P:D = C/(B-1) at 1K / 2K / 3K (LLaMA-13B)
  build
  timeout 1800 python tools/e2e_policies.py --model llama-13b --lengths 1024 --pd 1 2 5 10 15 20 30 50 \
    --policies sarathi request_level orca_best > gpurun_out/e2e_pd_c256.txt 2> gpurun_out/e2e_pd_c256.err
  timeout 1200 python tools/e2e_policies.py --model llama-13b --lengths 1024 --pd 1 2 5 10 15 20 30 50 --chunk 512 \
    --policies sarathi request_level > gpurun_out/e2e_pd_c512.txt 2> gpurun_out/e2e_pd_c512.err
  timeout 1500 python tools/e2e_policies.py --model llama-13b --lengths 1024 2048 3072 --pd-optimal \
    --policies sarathi request_level orca_best > gpurun_out/e2e_opt.txt 2> gpurun_out/e2e_opt.err
  ;;
kbcommit)
  # the k-block's empty-barrier commit inside the k-block asm block (SARATHI_GEMM_KBCOMMIT)
  build
  timeout 600 python -m pytest tests/test_gpu_gemm.py -x -q > gpurun_out/pytest_gemm.log 2>&1; echo rc=$? >> gpurun_out/pytest_gemm.log
  timeout 900 python -m pytest tests/test_gpu_model.py -x -q -k "not variants" > gpurun_out/pytest_model.log 2>&1; echo rc=$? >> gpurun_out/pytest_model.log
  for v in 1 0; do
    echo "== kbcommit=$v" >> gpurun_out/kbcommit.txt
    SARATHI_GEMM_KBCOMMIT=$v timeout 600 python tools/shard_step.py >> gpurun_out/kbcommit.txt 2>/dev/null
  done
  rm -rf gpurun_out/ab
  bash tools/ab.sh "SARATHI_GEMM_KBCOMMIT=1" "SARATHI_GEMM_KBCOMMIT=0"
  ;;
ksplit)
  # prefill key split on the TP-8 rank shapes after the session-3 GEMM changes (cost model vs forced)
  build
  for r in 1 2; do for k in 0 2 4 6 8; do
    echo "== r$r ksplit=$k" >> gpurun_out/ksplit.txt
    if [ $k = 0 ]; then timeout 600 python tools/shard_step.py --which llama70b-tp8 gpt3-tp8 >> gpurun_out/ksplit.txt 2>/dev/null
    else SARATHI_PREFILL_KSPLIT=$k timeout 600 python tools/shard_step.py --which llama70b-tp8 gpt3-tp8 >> gpurun_out/ksplit.txt 2>/dev/null; fi
  done; done
  ;;
*) echo "unknown experiment $exp" >&2; exit 2 ;;
esac
done
