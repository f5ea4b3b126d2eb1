# Horner-form derived legs A/B: int (mono ref), col (bi ref), h1 (all Horner), hmax2, hmax3
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv,noheader
SAR_LIB=tools/ab/libsar_h1.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
bash tools/gpu_sweep.sh "C3 C0 C2" tools/ab/libsar_int.so tools/ab/libsar_h1.so tools/ab/libsar_hmax2.so tools/ab/libsar_hmax3.so
bash tools/gpu_shard_sweep.sh C4 750 750 tools/ab/libsar_col.so tools/ab/libsar_h1.so tools/ab/libsar_hmax3.so
