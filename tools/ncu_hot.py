"""Per-instruction executed counts from an ncu report's source page (SASS), grouped into runs.

usage: python tools/ncu_hot.py REPORT.ncu-rep [min_fraction]
Prints the total warp instructions, then contiguous address ranges whose instructions execute
at the same count (basic blocks), with their share of all executed instructions and opcode mix."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
minf = float(sys.argv[2]) if len(sys.argv) > 2 else 0.005
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
# a multi-kernel report prints one table per kernel: keep the largest (the hot kernel's)
starts = [i for i, l in enumerate(lines) if l.startswith('"Address"')] + [len(lines)]
tables = []
for s0, s1 in zip(starts, starts[1:]):
    rs = [r for r in csv.DictReader(io.StringIO("\n".join(lines[s0:s1])))
          if (r.get("Instructions Executed") or "0").replace(",", "").isdigit()]
    tables.append(rs)
rows = max(tables, key=lambda rs: sum(int(r["Instructions Executed"] or 0) for r in rs))
tot = sum(int(r["Instructions Executed"] or 0) for r in rows)
print(f"total warp instructions {tot:.4e}")
blocks, cur = [], None
for r in rows:
    n = int(r["Instructions Executed"] or 0)
    op = r["Source"].strip()
    if op.startswith("@"):
        op = op.split(None, 1)[1]
    op = op.split()[0] if op else "?"
    if cur and cur["n"] == n:
        cur["ops"][op] += 1
        cur["end"] = r["Address"]
        cur["samples"] += int(r["Warp Stall Sampling (All Samples)"] or 0)
    else:
        cur = {"n": n, "start": r["Address"], "end": r["Address"], "ops": collections.Counter([op]),
               "samples": int(r["Warp Stall Sampling (All Samples)"] or 0)}
        blocks.append(cur)
totsamp = sum(b["samples"] for b in blocks) or 1
for b in blocks:
    k = sum(b["ops"].values())
    share = b["n"] * k / tot
    if share >= minf:
        print(f"{b['start'][-5:]}-{b['end'][-5:]} exec {b['n']:.3e} x {k:3d} = {share:6.1%}  samples {b['samples']/totsamp:6.1%}  "
              + " ".join(f"{o}:{c}" for o, c in b["ops"].most_common(12)))
