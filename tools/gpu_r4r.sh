timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_e2e.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/bench_e2e.json')); print(d['ms_per_step'], d['e2e']['ms_per_image'], d['roofline']['frac'])"
timeout 900 python tools/rank_probe2.py C3 8 2>&1 | grep -E '1-GPU|rebalanced x2'
