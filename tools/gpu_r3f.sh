# chirp-split waves vs BP DRAM traffic and time (C3, C0, C2): 8 / 16 / 32 (cur) waves
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv,noheader
bash tools/gpu_sweep.sh "C3 C0 C2" tools/ab/libsar_cur.so tools/ab/libsar_sw16.so tools/ab/libsar_sw8.so
for v in cur sw16 sw8; do
  SAR_LIB=tools/ab/libsar_$v.so timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"bp_kernel|split_sum|pair_kernel" --csv python tools/probe.py C3 > gpurun_out/dram_$v.csv 2>/dev/null
done
