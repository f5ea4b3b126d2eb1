# monostatic register floor (3 CTAs/SM) and derived-group unroll 4 / 7 vs cur
bash tools/gpu_sweep.sh "C3 C0 C2" tools/ab/libsar_cur.so tools/ab/libsar_mm3.so tools/ab/libsar_ju4.so tools/ab/libsar_ju7.so
