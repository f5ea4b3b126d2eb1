set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -x 2>&1 | tail -15
timeout 300 python tools/prof_shard.py C4 0 750 2 > gpurun_out/c4shard.log 2>&1; cat gpurun_out/c4shard.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bp_kernel -s 1 -c 1 -o gpurun_out/ncu_bp_bi_c4 python tools/prof_shard.py C4 0 750 2 > gpurun_out/ncu_c4.log 2>&1; echo ncu_rc=$?; tail -3 gpurun_out/ncu_c4.log
