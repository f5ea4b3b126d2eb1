timeout 900 ncu --set full --clock-control none --import-source on -k regex:bp_kernel -s 1 -c 1 -o gpurun_out/ncu_bp_bi_c4_r2 python tools/prof_shard.py C4 750 750 2 > gpurun_out/ncu_c4.log 2>&1; echo ncu_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bp_kernel -s 1 -c 1 -o gpurun_out/ncu_bp_c3_r2 python tools/prof_bp.py C3 2 > gpurun_out/ncu_c3.log 2>&1; echo ncu_rc=$?
python tools/probe.py C6p 2>&1 | grep "rc "
