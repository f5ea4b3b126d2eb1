# per-rank balance of both N > 1 legs (C3, C4) and the one-rank-group check of the N > 1 bench path, final build
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv,noheader
timeout 900 python tools/rank_probe2.py C3 2 4 8 2>&1 | tail -8
timeout 1500 python tools/rank_probe2.py C4 8 2>&1 | tail -4
timeout 900 python bench.py --all-legs --steps 3 --warmup 3 --no-cpu-baseline 2>gpurun_out/alllegs.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('all-legs C3', d['ms_per_step'], json.dumps(d.get('gather')))"
