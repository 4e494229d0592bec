"""SASS evidence of the production stage kernels (profiles/r2_sass_k_mm4.txt):
per kernel the instruction mix that shows the design (bulk copies UBLKCP,
mbarrier SYNCS, 128-bit pair loads/stores, FP64 FMAs, griddepcontrol) and an
excerpt of the paired-site gather round.  Run in the build container:
    python tools/sass_summary.py paper_1012_4382_b200/build/hb_mm4.o > profiles/r2_sass_k_mm4.txt"""
import re
import subprocess
import sys
from collections import Counter

obj = sys.argv[1]
names = subprocess.run(["cuobjdump", "-symbols", obj], capture_output=True, text=True).stdout
kernels = sorted(set(re.findall(r"(_ZN2hb5k_mm4IdLi7ELi2ELi\dELi1ELb0EEEvNS_7KParamsE)", names)))
if not kernels:
    kernels = sorted(set(re.findall(r"(_ZN2hb5k_mm4IdLi7ELi2ELi\d\w*KParamsE)", names)))
print("# cuobjdump -sass of k_mm4<double, 7, 2, stage> (config 4: d = 7, K + 1 = 2), sm_100a")
keys = ["LDG.E.128", "LDG.E.64", "LDG.E.64.CONSTANT", "LDG.E.128.CONSTANT", "STG.E.128", "STG.E.64",
        "UBLKCP", "SYNCS", "DFMA", "DADD", "DMUL", "LDS", "ACQBULK", "CCTL"]
for k in kernels:
    sass = subprocess.run(["cuobjdump", "-sass", "-fun", k, obj], capture_output=True, text=True).stdout
    ops = [l.split(";")[0].strip() for l in sass.splitlines() if re.match(r"\s+/\*[0-9a-f]{4}\*/", l)]
    mn = Counter(re.sub(r"^@!?U?P\w+\s+", "", o.split("*/", 1)[1].strip()).split(" ")[0] for o in ops)
    print(f"\n## {k}\ninstructions: {len(ops)}")
    for key in keys:
        n = sum(v for m, v in mn.items() if m == key or (m.startswith(key + ".") and key in ("SYNCS", "UBLKCP", "LDS")))
        if n:
            print(f"  {key:22s} {n}")
    other = [m for m in mn if m.startswith(("UBLKCP", "SYNCS", "ACQBULK", "UTMA"))]
    if other:
        print("  bulk/mbarrier mnemonics:", ", ".join(sorted(other)))
    if "Li4E" in k:  # an excerpt: the start of a gather round (128-bit loads)
        idx = [i for i, o in enumerate(ops) if "LDG.E.128.CONSTANT" in o]
        if idx:
            i0 = idx[len(idx) // 2]
            print("  excerpt (gather round, pair loads):")
            for o in ops[max(0, i0 - 4): i0 + 8]:
                print("    " + o.split("*/", 1)[1].strip())
