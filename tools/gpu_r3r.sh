# per-rank balance with equal tile counts vs calibrated tile-row weights (C3 2/4/8, C4 8)
timeout 900 python tools/rank_probe2.py C3 2 4 8 2>&1 | tail -14
timeout 1500 python tools/rank_probe2.py C4 8 2>&1 | tail -6
