# publish leg (SAR_SCATTER_PUBLISH): tests, per-rank probe, one-rank all-legs bench line
timeout 900 python -m pytest tests/test_gpu_scatter.py tests/test_bench_contract.py -q 2>&1 | tail -3
timeout 900 python tools/rank_probe2.py C3 2 8 2>&1 | grep -E '1-GPU|rebalanced x2'
timeout 900 python tools/rank_probe2.py C4 8 2>&1 | grep -E '1-GPU|rebalanced x2'
timeout 900 python bench.py --all-legs --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/alllegs.json 2>gpurun_out/alllegs.err; echo rc=$?
python -c "import json; d=json.load(open('gpurun_out/alllegs.json')); g=d['gather']; print(d['ms_per_step'], g['headline'], g['fused_ms'], g['publish_ms'], g['nccl_ms'], g['publish_check'])"
