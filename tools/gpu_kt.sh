# per-kernel durations (ncu launch list) of one probe run per build: bash tools/gpu_kt.sh CFG lib|pkgdir...
# writes gpurun_out/kt_<build>_<cfg>.csv; summarise with tools/kt_summary.py
cfg=$1; shift
mkdir -p gpurun_out
for lib in "$@"; do
  if [ -d "$lib" ]; then envs="SAR_PKG_ROOT=$lib"; else envs="SAR_LIB=$lib"; fi
  n=$(basename $lib .so)
  env $envs timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/kt_${n}_${cfg}.csv python tools/probe.py $cfg > /dev/null 2>&1
  echo "== $n rc=$?"
done
