# measured load balance (dist.rebalance) of both N > 1 legs, simulated rank by rank on one GPU; bench all-legs line
timeout 900 python tools/rank_probe2.py C3 2 4 8 2>&1 | tail -19
timeout 1500 python tools/rank_probe2.py C4 8 2>&1 | tail -7
timeout 900 python bench.py --all-legs --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/alllegs.json 2>gpurun_out/alllegs.err; echo rc=$?; wc -l gpurun_out/alllegs.json
