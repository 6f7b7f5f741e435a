# the paper's end-to-end policy comparison (§5.2) on the current kernels: LLaMA-33B and LLaMA-13B
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
P="sarathi request_level orca_best sarathi_b200"
timeout 1500 python tools/e2e_policies.py --model llama-33b --lengths 1024 2048 --pd 10 50 --policies $P > gpurun_out/e2e_33b.txt 2> gpurun_out/e2e_33b.err
timeout 1200 python tools/e2e_policies.py --model llama-13b --lengths 1024 --pd 1 10 50 --policies $P > gpurun_out/e2e_13b.txt 2> gpurun_out/e2e_13b.err
