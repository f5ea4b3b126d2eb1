# collinear legs A/B (int = previous commit, col = collinear groups/stages)
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv,noheader
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
bash tools/gpu_sweep.sh "C3 C0 C2" tools/ab/libsar_int.so tools/ab/libsar_col.so
bash tools/gpu_shard_sweep.sh C4 750 750 tools/ab/libsar_int.so tools/ab/libsar_col.so
