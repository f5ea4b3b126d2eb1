# usage: bash tools/gpu_sweep.sh "CFGS" lib... : bp timing of tuning builds (tools/probe.py), 2 rounds
cfgs=$1; shift
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv,noheader
# a directory argument is a whole package tree (e.g. a previous commit's build): SAR_PKG_ROOT
for rep in 1 2; do for lib in "$@"; do
  if [ -d "$lib" ]; then envs="SAR_PKG_ROOT=$lib"; else envs="SAR_LIB=$lib"; fi
  echo "== $(basename $lib) $(env $envs timeout 300 python tools/probe.py $cfgs 2>&1 | grep -E 'rc |Error|error' | sed 's/.*: rc/rc/' | tr '\n' ' ')"
done; done
