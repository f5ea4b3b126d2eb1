# derived-leg modes and per-chirp-leg equality (new test), then the bistatic configs
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv,noheader
SAR_LIB=paper_2306_09784_b200/libsar_check.so python tools/derive_modes.py
timeout 900 python -m pytest tests/test_gpu_derived.py -q 2>&1 | tail -15
