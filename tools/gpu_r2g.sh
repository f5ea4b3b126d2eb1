python tools/dbg_derive.py 2>&1 | head -2
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 2>&1 | tail -3
bash tools/gpu_sweep.sh "C3 C0 C2 C6 C6p" tools/variants/libsar_der3.so
bash tools/gpu_shard_sweep.sh C4 750 750 tools/variants/libsar_der3.so
