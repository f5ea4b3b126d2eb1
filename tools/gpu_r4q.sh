# pair-row window per chirp chunk: 20 / 40 (default) / 80 / 160 MB on C4 full, C4 rank shard, C3
for w in 20 40 80 160; do
  echo "window $w MB: $(SAR_BP_L2_WINDOW_MB=$w timeout 300 python tools/probe.py C4 C3 2>&1 | grep -E 'rc ' | sed 's/.*: rc/rc/' | tr '\n' ' ') shard $(SAR_BP_L2_WINDOW_MB=$w timeout 300 python tools/prof_shard.py C4 750 750 3 2>&1 | tail -1)"
done
