# scatter family at 3 CTAs/SM too (mm3c), per-rank fused leg N = 2/4/8; scatter waves 8 / 32
for lib in mm3c; do SAR_LIB=tools/ab/libsar_$lib.so timeout 900 python tools/rank_probe2.py C3 2 4 8 2>&1 | grep -E '1-GPU|rebalanced x2'; done
for w in 8 32; do echo "scatter waves $w"; SAR_BP_SCATTER_WAVES=$w SAR_LIB=tools/ab/libsar_mm3c.so timeout 900 python tools/rank_probe2.py C3 8 2>&1 | grep -E 'rebalanced x2: fused'; done
