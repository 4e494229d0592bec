"""Attribute ncu SASS-level stall samples to CUDA source lines.

    python tools/sass_lines.py <cubin-disasm-with-g.txt> <kernel-mangled-name> <ncu-source-sass.csv> [src_dir]
(the disassembly comes from `nvdisasm -g` of the cubin extracted with `cuobjdump -xelf`)."""
import csv
import re
import sys
from pathlib import Path


def main():
    dis, name, csvf = sys.argv[1:4]
    src_dir = Path(sys.argv[4]) if len(sys.argv) > 4 else Path("paper_1012_4382_b200/csrc")
    txt = open(dis).read().split("\n")
    start = next(i for i, l in enumerate(txt) if l.startswith(name + ":"))
    end = next((i for i in range(start + 2, len(txt)) if txt[i].startswith(".text.")), len(txt))
    addr2line, cur = {}, None
    for l in txt[start:end]:
        m = re.search(r'//## File "(.*)", line (\d+)', l)
        if m:
            cur = (Path(m.group(1)).name, int(m.group(2)))
            continue
        m = re.search(r"/\*([0-9a-f]{4,})\*/", l)
        if m and cur:
            addr2line[int(m.group(1), 16)] = cur
    rows = list(csv.reader(open(csvf)))
    base = int(rows[2][0], 16)
    agg, tot = {}, 0
    for r in rows[2:]:
        try:
            a, s = int(r[0], 16) - base, int(float(r[2] or 0))
        except (ValueError, IndexError):
            continue
        k = addr2line.get(a, ("?", 0))
        agg[k] = agg.get(k, 0) + s
        tot += s
    print(f"samples {tot}")
    for (f, ln), s in sorted(agg.items(), key=lambda x: -x[1])[:30]:
        p = src_dir / f
        text = p.read_text().split("\n")[ln - 1].strip()[:90] if ln and p.exists() else ""
        print(f"{f}:{ln:5d} {100 * s / tot:5.1f}%  {text}")


if __name__ == "__main__":
    main()
