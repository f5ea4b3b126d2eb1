# 16 x 32 range-compression sub-transform (w16, default) vs Stockham (cur): parity + timing
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "rc_ or largest_fft" 2>&1 | tail -3
bash tools/gpu_sweep.sh "C3 C2 C4" tools/ab/libsar_cur.so tools/ab/libsar_w16.so
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rc_kernel_warp -s 2 -c 1 -o gpurun_out/ncu_rc16 -f python tools/probe.py C3 > gpurun_out/ncu_rc16.log 2>&1; echo rc=$?
