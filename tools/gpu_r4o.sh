# split chunks bounded by the pair-row window in L2 (l2w) vs cur: C4 shard DRAM + time, configs
for lib in cur l2w; do
  SAR_LIB=tools/ab/libsar_$lib.so timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:bp_kernel_bi -s 1 -c 1 python tools/prof_shard.py C4 750 750 2 2>&1 | grep -E 'dram__|gpu__time' | sed "s/^/$lib /"
done
bash tools/gpu_shard_sweep.sh C4 750 750 tools/ab/libsar_cur.so tools/ab/libsar_l2w.so
bash tools/gpu_sweep.sh "C3 C0 C2 C6" tools/ab/libsar_cur.so tools/ab/libsar_l2w.so
