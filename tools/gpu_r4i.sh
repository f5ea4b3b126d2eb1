# bistatic at three CTAs per SM (b3), with Horner 3/4 terms (b3h); Horner 3-term at four CTAs (b4h3); C4 shard + C6
bash tools/gpu_shard_sweep.sh C4 750 750 tools/ab/libsar_cur.so tools/ab/libsar_b3.so tools/ab/libsar_b3h.so tools/ab/libsar_b4h3.so
bash tools/gpu_sweep.sh "C6" tools/ab/libsar_cur.so tools/ab/libsar_b3.so tools/ab/libsar_b3h.so tools/ab/libsar_b4h3.so
for cb in 32 40; do echo "b3 cb=$cb"; SAR_BP_SHAPE=8,4,0,$cb bash tools/gpu_shard_sweep.sh C4 750 750 tools/ab/libsar_b3.so | head -1; done
