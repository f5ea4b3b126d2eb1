# collinear RX records as one float4 {s, c, nM, address} (rec) vs the previous build (cur)
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv,noheader
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "bistatic or rx or mimo or C4 or full_size" 2>&1 | tail -3
bash tools/gpu_shard_sweep.sh C4 750 750 tools/ab/libsar_cur.so tools/ab/libsar_rec.so
bash tools/gpu_sweep.sh "C6" tools/ab/libsar_cur.so tools/ab/libsar_rec.so
