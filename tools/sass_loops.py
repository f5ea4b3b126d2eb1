"""List the backward-branch loops of one kernel's SASS that contain MUFU, with their instruction mix.

usage: python tools/sass_loops.py LIB.so NAME_SUBSTRING [NAME_SUBSTRING2]"""
import collections
import re
import subprocess
import sys

lib, keys = sys.argv[1], sys.argv[2:]
txt = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
for f in re.split(r"\n\s+Function : ", txt):
    name = f.split("\n", 1)[0]
    if not all(k in name for k in keys):
        continue
    ins = []
    for line in f.split("\n"):
        m = re.search(r"/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if m:
            ins.append((int(m.group(1), 16), m.group(2).strip()))
    idx = {a: i for i, (a, _) in enumerate(ins)}
    print(name[:120], len(ins), "instructions")
    for i, (a, t) in enumerate(ins):
        m = re.search(r"BRA(?:\.U)?\s+(?:!?U?P\d, )?0x([0-9a-f]+)", t)
        if not m:
            continue
        tgt = int(m.group(1), 16)
        if tgt >= a or tgt not in idx:
            continue
        body = ins[idx[tgt]: i + 1]
        ops = collections.Counter()
        for _, x in body:
            x = re.sub(r"^@!?U?P\w+\s+", "", x)
            ops[x.split()[0]] += 1
        if any(k.startswith("MUFU") for k in ops):
            print(f"  loop {tgt:#x}-{a:#x}: {len(body)} instr", dict(ops.most_common()))
