# evidence after the bistatic stage changes: tests, smoke, bench lines, launch list, full capture of C3 and of the C4 rank shard
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
SAR_LIB=paper_2306_09784_b200/libsar_check.so timeout 900 python tools/check_cases.py > gpurun_out/check_cases.log 2>&1; echo check_rc=$?; tail -3 gpurun_out/check_cases.log
bash tools/gpu_evidence_all.sh
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bp_kernel_bi -s 1 -c 1 -o gpurun_out/ncu_bi_c4 -f python tools/prof_shard.py C4 750 750 2 > gpurun_out/ncu_bi_c4.log 2>&1; echo bi_rc=$?
