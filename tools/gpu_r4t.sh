# sar_form_image banded readback pipeline: e2e of C3 / C4 with 0 (epilogue host stores), 2, 4, 8 bands; tests with 4
for nb in 0 2 4 8; do
  SAR_FORM_BANDS=$nb timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b_$nb.json 2>/dev/null
  echo "bands $nb: $(python -c "import json; d=json.load(open('gpurun_out/b_$nb.json')); print(d['ms_per_step'], d['e2e']['ms_per_image'])")"
done
for nb in 0 4; do SAR_FORM_BANDS=$nb timeout 900 python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b4_$nb.json 2>/dev/null; echo "C4 bands $nb: $(python -c "import json; d=json.load(open('gpurun_out/b4_$nb.json')); print(d['ms_per_step'], d['e2e']['ms_per_image'])")"; done
SAR_FORM_BANDS=4 timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "form_image" 2>&1 | tail -2
