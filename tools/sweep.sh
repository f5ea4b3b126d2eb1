# BP CTA-shape / ring sweep (SAR_BP_SHAPE = ncw,pb,stages,chirps_per_stage)
cfg=${1:-C3}; shift
for sh in ${@:-"8,4,0,0" "4,8,0,0" "4,8,4,16" "4,8,3,16" "4,8,6,8" "4,4,0,0" "4,4,4,16" "4,4,8,16" "8,8,0,0"}; do
  echo "== $sh $(SAR_BP_SHAPE=$sh timeout 120 python tools/probe.py $cfg 2>&1 | grep -E 'rc |Error|error')"
done
