python tools/check_cases.py 2>&1 | tail -3
SAR_BP_DERIVE=0 timeout 300 python tools/probe.py C3 C0 2>&1 | grep "rc "
bash tools/gpu_sweep.sh "C3 C0 C2" tools/variants/libsar_der.so tools/variants/libsar_derm4.so tools/variants/libsar_derm3.so
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "full_size or C1 or small_scenes or translation or permutation or near_field or shards or split" 2>&1 | tail -3
