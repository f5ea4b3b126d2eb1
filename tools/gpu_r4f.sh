# 3-CTA monostatic default with 64 KB ring budget; scatter family at 4 CTAs
bash tools/gpu_sweep.sh "C3 C0 C2 C6" tools/ab/libsar_cur.so tools/ab/libsar_mm3b.so
timeout 900 python tools/rank_probe2.py C3 8 2>&1 | tail -7
