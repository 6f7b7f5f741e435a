# paper experiments re-run on the round-2 kernels: end-to-end policies (33B, 13B) and the decode sweep
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 python tools/e2e_policies.py --model llama-33b --lengths 1024 2048 --pd 10 50 --policies sarathi request_level orca_best sarathi_b200 > gpurun_out/e2e_33b.txt 2> gpurun_out/e2e_33b.err
timeout 1200 python tools/e2e_policies.py --model llama-13b --lengths 1024 --pd 1 10 50 --policies sarathi request_level orca_best sarathi_b200 > gpurun_out/e2e_13b.txt 2> gpurun_out/e2e_13b.err
timeout 900 python tools/decode_sweep.py > gpurun_out/decode_sweep.txt 2> gpurun_out/decode_sweep.err
