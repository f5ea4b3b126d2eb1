# on top of 3 CTAs/SM (mm3): 3-term Horner, collinear monostatic groups, 16-chirp groups, 48 chirps per stage
bash tools/gpu_sweep.sh "C3 C0 C2" tools/ab/libsar_mm3.so tools/ab/libsar_mm3h3.so tools/ab/libsar_mm3col.so tools/ab/libsar_mm3g16.so
echo "cb 48"; SAR_BP_SHAPE=8,4,0,48 bash tools/gpu_sweep.sh "C3 C2" tools/ab/libsar_mm3.so
