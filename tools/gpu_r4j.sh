# bistatic at three CTAs with Horner stages: GPU tests, bistatic bench lines, C4 per-rank balance
timeout 1500 python -m pytest tests -m gpu -q --timeout 1200 > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_gpu.log
mkdir -p gpurun_out/configs
for c in C4 C6 C6p; do timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/configs/bench_$c.json 2> gpurun_out/configs/bench_$c.err; echo $c rc=$?; done
timeout 1500 python tools/rank_probe2.py C4 8 2>&1 | grep -E '1-GPU|rebalanced x2'
