for cfg in "32 7" "32 100" "8 100" "16 100" "8 7" "4 100"; do set -- $cfg
  echo "== scatter waves $1 unsplit $2"; SAR_BP_SCATTER_WAVES=$1 SAR_BP_SCATTER_UNSPLIT=$2 python tools/rank_probe2.py C3 2 8 2>&1 | grep fused
done
