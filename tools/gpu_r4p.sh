# L2-window split on whole images (C4 full: 35344 tiles) vs no window (now)
bash tools/gpu_sweep.sh "C4 C3" tools/ab/libsar_cur.so tools/ab/libsar_now.so
for lib in cur now; do
  SAR_LIB=tools/ab/libsar_$lib.so timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"bp_kernel|split_sum" -s 2 -c 2 python tools/probe.py C4 2>&1 | grep -E 'dram__|gpu__time|split_sum|bp_kernel' | sed "s/^/$lib /"
done
