bash tools/gpu_sweep.sh "C3 C0" tools/ab/libsar_cur.so tools/ab/libsar_mm2.so
for cb in 16 20 32; do echo "bi cb=$cb"; SAR_BP_SHAPE=8,4,0,$cb bash tools/gpu_shard_sweep.sh C4 750 750 tools/ab/libsar_cur.so | head -1; done
echo "bi default"; bash tools/gpu_shard_sweep.sh C4 750 750 tools/ab/libsar_cur.so | head -1
