# usage: bash tools/gpu_shard_sweep.sh CFG ROW0 NROW lib...   (bp ms of one row shard per build, 2 rounds)
cfg=$1; r0=$2; n=$3; shift 3
for rep in 1 2; do for lib in "$@"; do
  if [ -d "$lib" ]; then envs="SAR_PKG_ROOT=$lib"; else envs="SAR_LIB=$lib"; fi
  echo "== $(basename $lib) $(env $envs timeout 300 python tools/prof_shard.py $cfg $r0 $n 3 2>&1 | tail -1)"
done; done
