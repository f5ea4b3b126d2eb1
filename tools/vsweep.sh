# usage: bash tools/vsweep.sh CFG lib:shape [lib:shape ...]   (timing of library variants x CTA shapes)
cfg=$1; shift
for ls in "$@"; do lib=${ls%%:*}; sh=${ls##*:}
  echo "== $lib $sh $(SAR_LIB=$lib SAR_BP_SHAPE=$sh timeout 120 python tools/probe.py $cfg 2>&1 | grep -E 'rc |Error|error')"
done
