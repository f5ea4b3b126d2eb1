# usage: bash tools/libsweep.sh "CFG..." lib [lib ...]   (bp/rc timing of tuning builds, default shape)
cfgs=$1; shift
for rep in 1 2; do for lib in "$@"; do
  echo "== $lib $(SAR_LIB=$lib timeout 300 python tools/probe.py $cfgs 2>&1 | grep -E 'rc |Error|error' | sed 's/.*: rc/rc/' | tr '\n' ' ')"
done; done
