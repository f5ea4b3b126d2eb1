timeout 300 python tools/probe.py C3 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rc_kernel_warp -s 2 -c 1 -o gpurun_out/ncu_rc -f python tools/probe.py C3 > gpurun_out/ncu_rc.log 2>&1; echo rc=$?
