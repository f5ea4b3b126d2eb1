bash tools/gpu_sweep.sh "C3 C0" tools/variants/libsar_der6.so
SAR_BP_SHAPE=4,8 bash tools/gpu_sweep.sh "C3 C0" tools/variants/libsar_der6.so
SAR_BP_SHAPE=8,8 bash tools/gpu_sweep.sh "C3 C0" tools/variants/libsar_der6.so
bash tools/gpu_shard_sweep.sh C4 750 750 tools/variants/libsar_der6.so tools/variants/libsar_der6b3.so
