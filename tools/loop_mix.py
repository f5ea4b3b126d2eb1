"""Instruction mix of bp_kernel's monostatic consumer chirp loop (the basic block holding
MUFU.RSQ) in a libsar build: python tools/loop_mix.py [lib] [kernel-substring]."""
import collections, re, subprocess, sys, tempfile, os

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2306_09784_b200/libsar.so"
kern = sys.argv[2] if len(sys.argv) > 2 else "bp_kernel_monoILb0ELb0ELi8ELi4E"
with tempfile.TemporaryDirectory() as d:
    subprocess.run(["cuobjdump", "-xelf", "bp_kernel.sm_100a.cubin", os.path.abspath(lib)], cwd=d, check=True,
                   capture_output=True)
    sass = subprocess.run(["cuobjdump", "-sass", "bp_kernel.sm_100a.cubin"], cwd=d, check=True,
                          capture_output=True, text=True).stdout
fn = sass.split("Function : ")
body = next(f for f in fn if kern in f.split("\n")[0])
ins = [l for l in body.split("\n") if re.search(r"/\*[0-9a-f]{4}\*/", l)]
addr = lambda l: int(re.search(r"/\*([0-9a-f]{4,})\*/", l).group(1), 16)
i_rsq = next(i for i, l in enumerate(ins) if re.search(r"MUFU\.RSQ R", l))
# loop = from the target of the backward branch after the first RSQ to that branch
j = next(j for j in range(i_rsq, len(ins)) if re.search(r"BRA 0x([0-9a-f]+)", ins[j]) and
         int(re.search(r"BRA 0x([0-9a-f]+)", ins[j]).group(1), 16) < addr(ins[i_rsq]))
tgt = int(re.search(r"BRA 0x([0-9a-f]+)", ins[j]).group(1), 16)
i0 = next(i for i, l in enumerate(ins) if addr(l) == tgt)
loop = ins[i0:j + 1]
mix = collections.Counter(re.sub(r"^\s*/\*[0-9a-f]+\*/\s*(@!?U?P\d\s+)?", "", l).split()[0] for l in loop)
print(f"{kern}: {len(loop)} instructions in the chirp loop")
for k, v in sorted(mix.items(), key=lambda kv: -kv[1]):
    print(f"  {v:3d} {k}")
