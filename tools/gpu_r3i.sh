# bistatic A/B on the C4 rank shard: compile-time 4 RX, RX unroll 2, chirps per stage 4 / 16 (SAR_BP_SHAPE)
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv,noheader
bash tools/gpu_shard_sweep.sh C4 750 750 tools/ab/libsar_cur.so tools/ab/libsar_nrx4.so tools/ab/libsar_rxu2.so
for cb in 4 16; do echo "cb=$cb"; SAR_BP_SHAPE=8,4,0,$cb bash tools/gpu_shard_sweep.sh C4 750 750 tools/ab/libsar_cur.so; done
