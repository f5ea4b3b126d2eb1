# A/B: bistatic 4x4 (polar C6p) register floor; monostatic derived group size 16 / 4 with the new tails
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv,noheader
bash tools/gpu_sweep.sh "C6p" tools/ab/libsar_cur.so tools/ab/libsar_bs4.so tools/ab/libsar_bs6.so
bash tools/gpu_sweep.sh "C3 C0 C2" tools/ab/libsar_cur.so tools/ab/libsar_g16.so tools/ab/libsar_g16u.so tools/ab/libsar_g4.so
