# default 3 CTAs/SM monostatic: C0 ring shapes, C5 frames, per-rank scatter balance
for sh in 8,4,0,24 8,4,0,32 8,4,3,24 8,4,0,16; do echo "C0 shape $sh: $(SAR_BP_SHAPE=$sh timeout 300 python tools/probe.py C0 2>&1 | grep -E 'rc |rror' | sed 's/.*: rc/rc/')"; done
echo "C3 shape 8,4,4,32: $(SAR_BP_SHAPE=8,4,4,32 timeout 300 python tools/probe.py C3 2>&1 | grep -E 'rc |rror' | sed 's/.*: rc/rc/')"
echo "C3 shape 8,4,2,32: $(SAR_BP_SHAPE=8,4,2,32 timeout 300 python tools/probe.py C3 2>&1 | grep -E 'rc |rror' | sed 's/.*: rc/rc/')"
timeout 900 python tools/rank_probe2.py C3 8 2>&1 | tail -7
