# C4 rank shard DRAM traffic vs chirps per stage (16 default, 24)
for cb in 16 24; do
  SAR_BP_SHAPE=8,4,0,$cb timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:bp_kernel_bi -s 1 -c 1 python tools/prof_shard.py C4 750 750 2 2>&1 | grep -E 'dram__|gpu__time|hit_rate' | sed "s/^/cb=$cb /"
done
