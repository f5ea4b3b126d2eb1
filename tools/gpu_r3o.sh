# polar 4 x 4 bistatic shape with derived stages (C6p)
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv,noheader
bash tools/gpu_sweep.sh "C6p" tools/ab/libsar_cur.so tools/ab/libsar_d44.so tools/ab/libsar_d44m3.so
SAR_LIB=tools/ab/libsar_d44.so timeout 900 python -m pytest tests/test_gpu_polar.py -x -q 2>&1 | tail -2
