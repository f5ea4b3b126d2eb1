# C6p (polar, 8 RX) shape / chirps-per-stage sweep
bash tools/gpu_sweep.sh C6p tools/ab/libsar_cur.so | head -2
for sh in 4,4,0,1 4,4,0,3 4,4,0,4 4,4,0,6 8,4,0,2 8,4,0,4 4,8,0,2 4,8,0,4; do echo "shape $sh: $(SAR_BP_SHAPE=$sh SAR_LIB=tools/ab/libsar_cur.so timeout 300 python tools/probe.py C6p 2>&1 | grep -E 'rc |rror' | sed 's/.*: rc/rc/')"; done
