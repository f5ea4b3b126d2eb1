nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv,noheader
SAR_LIB=paper_2306_09784_b200/libsar_check.so python tools/derive_modes.py
timeout 900 python -m pytest tests/test_gpu_derived.py -q -s 2>&1 | grep -E 'derived vs|passed|failed|Error|assert|\{' | head -30
echo "== previous round-2 build (7165a91)"
SAR_LIB=tools/ab/libsar_r2.so timeout 900 python -m pytest tests/test_gpu_derived.py -q -s -k equals 2>&1 | grep -E 'derived vs|passed|failed' | head -30
