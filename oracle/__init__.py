"""fp64 CPU oracle for the SARATHI hybrid-batch forward pass (arXiv 2308.16369).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import anything under
``oracle/``.  The product path (``paper_2308_16369_b200``) never imports it and shares no
code with it; the only common dependency is the seeded input generator ``synth``, which
holds none of the method's arithmetic.

Modules
  model    -- the plain causal-LM forward (per request, whole history, no cache, no chunking)
              and the incremental replay of a hybrid-batch schedule with an fp64 KV cache.
  sched    -- decode-maximal batching scheduler, chunk planning, block allocator and
              slot mapping, paper formulas (max batch size, P:D balance, tile adjustment).
  metrics  -- the paper's throughput metrics (marginal decode time etc.).

Citations: ``P:Lnnn`` = /root/reference/PAPER.md line nnn (section noted), ``S:Lnnn`` =
SPEC.md line nnn.  Where the paper is silent the reading number (O-n) refers to the table in
DESIGN.md §3.

Parity status: every function here is pinned by a ``-m "not gpu"`` test in
``tests/test_oracle_*.py`` (HF LlamaForCausalLM fp64, closed forms, brute force, paper
arithmetic).  The GELU-tanh FFN variant has no library twin; it is pinned by its closed form
(torch.nn.functional.gelu(approximate="tanh")) plus the shared norm/attention path.
"""
