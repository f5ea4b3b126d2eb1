# pair-row window 40 (default) / 56 / 64 MB: C3, C4 full, C4 rank shard time; C3 DRAM
for w in 40 56 64; do
  echo "window $w MB: $(SAR_BP_L2_WINDOW_MB=$w timeout 300 python tools/probe.py C3 C4 2>&1 | grep -E 'rc ' | sed 's/.*: rc/rc/' | tr '\n' ' ') shard $(SAR_BP_L2_WINDOW_MB=$w timeout 300 python tools/prof_shard.py C4 750 750 3 2>&1 | tail -1)"
  SAR_BP_L2_WINDOW_MB=$w timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"bp_kernel|split_sum" -s 2 -c 2 python tools/probe.py C3 2>&1 | grep -E 'dram__' | sed "s/^/  w=$w /"
done
