set -x
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -x 2>&1 | tail -4
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c3.log 2>&1; echo bench_rc=$?; tail -c 2500 gpurun_out/bench_c3.log
timeout 300 python bench.py --gpus 2 --steps 2 --warmup 3 2>&1 | tail -2
