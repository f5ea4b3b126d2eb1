# bistatic: compile-time 4 RX x chirps per stage (C4 shard), C6 (8 RX) chirps per stage
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv,noheader
for cb in 8 12 16 24; do echo "cb=$cb"; SAR_BP_SHAPE=8,4,0,$cb bash tools/gpu_shard_sweep.sh C4 750 750 tools/ab/libsar_nrx4.so; done
for cb in 4 6 8; do echo "C6 cb=$cb"; SAR_BP_SHAPE=8,4,0,$cb bash tools/gpu_sweep.sh C6 tools/ab/libsar_cur.so; done
