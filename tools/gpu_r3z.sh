# C0 (1201^2 at 2.5 cm: W = 59, near-field first rows) shape / ring sweep
bash tools/gpu_sweep.sh C0 tools/ab/libsar_cur.so | head -2
for sh in 8,4,0,8 8,4,0,24 8,4,3,16 8,4,2,16 4,4,0,16 4,4,0,32 4,8,0,16; do echo "shape $sh: $(SAR_BP_SHAPE=$sh SAR_LIB=tools/ab/libsar_cur.so timeout 300 python tools/probe.py C0 2>&1 | grep -E 'rc |rror' | sed 's/.*: rc/rc/')"; done
