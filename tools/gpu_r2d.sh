set -x
timeout 2400 python -m pytest tests -m gpu -q --timeout 1200 -x --durations=8 2>&1 | tail -16
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1; echo bench_rc=$?; tail -c 1500 gpurun_out/bench_c3.log
