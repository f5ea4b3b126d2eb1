run() { echo "== $1 $2 $(SAR_LIB=$1 SAR_BP_SHAPE=$2 timeout 120 python tools/probe.py ${3:-C3} 2>&1 | grep -E 'rc |Error|error')"; }
run paper_2306_09784_b200/libsar.so 4,8,0,0
run tools/variants/libsar_mb48_6.so 4,8,4,16
run tools/variants/libsar_mb48_6.so 4,8,3,16
run tools/variants/libsar_mb48_7.so 4,8,3,16
run tools/variants/libsar_mb84_5.so 8,4,4,16
run tools/variants/libsar_mb84_5.so 8,4,3,16
