# bistatic register budget A/B (3 CTAs/SM, +Horner) and an ncu capture of the current bistatic kernel
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv,noheader
bash tools/gpu_shard_sweep.sh C4 750 750 tools/ab/libsar_cur.so tools/ab/libsar_bi3.so tools/ab/libsar_bi3h.so tools/ab/libsar_h1.so
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bp_kernel_bi -s 1 -c 1 -o gpurun_out/ncu_bi_cur -f python tools/prof_shard.py C4 750 750 2 > gpurun_out/ncu_bi_cur.log 2>&1
SAR_LIB=tools/ab/libsar_h1.so timeout 600 ncu --set full --clock-control none --import-source on -k regex:bp_kernel_bi -s 1 -c 1 -o gpurun_out/ncu_bi_h1 -f python tools/prof_shard.py C4 750 750 2 > gpurun_out/ncu_bi_h1.log 2>&1
