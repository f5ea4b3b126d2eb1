# monostatic chirps per stage in steps of the derived group (cb) vs halving (cur)
bash tools/gpu_sweep.sh "C0 C3 C2" tools/ab/libsar_cur.so tools/ab/libsar_cb.so
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "full_size or cta_shapes or C1" 2>&1 | tail -2
