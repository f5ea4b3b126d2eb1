set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 -x 2>&1 | tail -25
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench1.log 2>&1; echo bench_rc=$?; tail -3 gpurun_out/bench1.log
timeout 300 python tools/prof_bp.py C3 2 > gpurun_out/plain_prof.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:bp_kernel -s 1 -c 1 -o gpurun_out/prof_bp_c3 python tools/prof_bp.py C3 2 > gpurun_out/ncu_full.log 2>&1; echo ncu_rc=$?; tail -3 gpurun_out/ncu_full.log
