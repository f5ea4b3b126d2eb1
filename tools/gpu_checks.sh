# bounds-check build over every kernel family (compute-sanitizer is closed on this pool)
SAR_LIB=paper_2306_09784_b200/libsar_check.so timeout 900 python tools/check_cases.py 2>&1 | tee gpurun_out/check_cases.log | tail -20
