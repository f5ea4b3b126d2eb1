# evidence of the session-3 build: bounds-check cases, then the round evidence (tests, smoke, bench lines, launch list, full capture)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
SAR_LIB=paper_2306_09784_b200/libsar_check.so timeout 900 python tools/check_cases.py > gpurun_out/check_cases.log 2>&1; echo check_rc=$?; tail -3 gpurun_out/check_cases.log
bash tools/gpu_evidence_all.sh
