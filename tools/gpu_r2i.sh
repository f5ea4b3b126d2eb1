bash tools/gpu_sweep.sh "C3 C0 C6 C6p" tools/variants/libsar_der5.so tools/variants/libsar_nodb.so tools/variants/libsar_nodm.so tools/variants/old_pkg
bash tools/gpu_shard_sweep.sh C4 750 750 tools/variants/libsar_der5.so tools/variants/libsar_nodb.so
