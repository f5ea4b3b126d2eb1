set -x
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -x 2>&1 | tail -15
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c3.log 2>&1; echo bench_rc=$?; tail -c 3000 gpurun_out/bench_c3.log
timeout 300 python tools/rank_probe.py > gpurun_out/rank_probe.log 2>&1; cat gpurun_out/rank_probe.log
