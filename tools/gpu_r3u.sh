# rc_kernel_warp timing experiments (wrong values): what each memory stream costs
for v in cur rc1 rc2 rc4 rc8 rc15; do echo "== $v $(SAR_LIB=tools/ab/libsar_$v.so timeout 300 python tools/probe.py C3 2>&1 | grep -E 'rc ' | sed 's/.*: rc/rc/')"; done
for v in cur rc15; do echo "== $v $(SAR_LIB=tools/ab/libsar_$v.so timeout 300 python tools/probe.py C3 2>&1 | grep -E 'rc ' | sed 's/.*: rc/rc/')"; done
