PROBE_PLAIN_TILES=1 timeout 900 python tools/rank_probe2.py C3 2 8 2>&1 | grep -E '1-GPU|it2|rebalanced x2: fused'
