# banded readback only for grids that fill the GPU twice per band: e2e of every config
for c in C3 C2 C0 C4 C6 C6p; do timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/be_$c.json 2>/dev/null; echo "$c $(python -c "import json; d=json.load(open('gpurun_out/be_$c.json')); print(d['ms_per_step'], d['e2e']['ms_per_image'])")"; done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "form_image" 2>&1 | tail -1
