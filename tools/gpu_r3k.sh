# bistatic auto chirps-per-stage + compile-time 4 RX (new) vs previous (cur, nrx4); monostatic cb sweep
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_polar.py tests/test_gpu_scatter.py -x -q 2>&1 | tail -3
bash tools/gpu_shard_sweep.sh C4 750 750 tools/ab/libsar_nrx4.so tools/ab/libsar_new.so
bash tools/gpu_sweep.sh "C6 C6p" tools/ab/libsar_cur.so tools/ab/libsar_new.so
for cb in 16 48 64; do echo "mono cb=$cb"; SAR_BP_SHAPE=8,4,0,$cb bash tools/gpu_sweep.sh "C3 C0" tools/ab/libsar_cur.so; done
