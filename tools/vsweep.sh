# timing of library variants x shapes on C3
for lib in paper_2306_09784_b200/libsar.so tools/variants/libsar_u2.so tools/variants/libsar_u4.so; do
 for sh in "8,4,0,0" "4,8,0,0" "4,4,4,16"; do
  echo "== $lib $sh $(SAR_LIB=$lib SAR_BP_SHAPE=$sh timeout 120 python tools/probe.py ${1:-C3} 2>&1 | grep -E 'rc |Error|error')"
 done
done
