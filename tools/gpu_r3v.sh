# range compression: stage twiddles from register bases + ramp recurrence (rcnew) vs cur; MINB 4
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "rc_ or largest_fft" 2>&1 | tail -2
bash tools/gpu_sweep.sh "C3 C2 C4" tools/ab/libsar_cur.so tools/ab/libsar_rcnew.so tools/ab/libsar_rcm4.so
