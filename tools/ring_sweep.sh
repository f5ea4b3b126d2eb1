# usage: bash tools/ring_sweep.sh CFG "shape..."  (SAR_BP_SHAPE=ncw,pb,stages,cb ring / CTA-shape overrides)
cfg=$1; shift
for rep in 1 2; do for sh in $@; do
  echo "== $sh $(SAR_BP_SHAPE=$sh timeout 300 python tools/probe.py $cfg 2>&1 | grep 'rc ' | sed 's/.*: rc/rc/')"
done; done
