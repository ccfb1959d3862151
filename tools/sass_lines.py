"""Warp-stall samples of an ncu SASS source export aggregated by CUDA source line.

    python tools/sass_lines.py <export.source.csv> <object.o> [top]

The export is `ncu -i R --page source --csv` (SASS view, one row per instruction in address
order); the object is the in-tree build of the same kernel (nvdisasm -g line info).  The
kernel is matched by its demangled name in the export's first row."""
import collections
import csv
import os
import re
import subprocess
import sys
import tempfile


def main(exp, obj, top=40):
    rows = list(csv.reader(open(exp)))
    kname = rows[0][1]
    h = rows[1]
    data = rows[2:]
    si = h.index("Warp Stall Sampling (All Samples)")
    # template args of the demangled name -> the mangled "ILi16ELi4ELb0..." pattern
    m = re.search(r"(\w+)<(\([^>]*)>\(", kname)
    base, targs = m.group(1), m.group(2)
    parts = []
    for a in targs.split(","):
        m = re.match(r"\s*\((\w+)\)(-?\d+)", a)
        parts.append(("Lb" if m.group(1) == "bool" else "Li") + m.group(2) + "E")
    pat = base + "I" + "".join(parts) + "E"
    with tempfile.TemporaryDirectory() as d:
        subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
        cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
        sass = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cub)], capture_output=True, text=True).stdout
    lines = sass.splitlines()
    start = [i for i, l in enumerate(lines) if l.startswith("_Z") and pat in l and l.endswith(":")][0]
    loc = {}
    cur = None
    for l in lines[start + 1:]:
        if l.startswith(".text.") or (l.startswith("_Z") and l.endswith(":")):
            break
        m = re.match(r'\s*//## File "(.*)", line (\d+)', l)
        if m:
            cur = (os.path.basename(m.group(1)), int(m.group(2)))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
        if m:
            loc[int(m.group(1), 16)] = cur
    agg = collections.Counter()
    tot = 0.0
    for i, r in enumerate(data):
        try:
            v = float(r[si] or 0)
        except ValueError:
            continue
        tot += v
        agg[loc.get(16 * i)] += v
    src = {}
    print(f"# {kname[:120]}\n# {len(data)} instructions, {tot:.0f} samples")
    for (key, v) in agg.most_common(top):
        if key is None:
            print(f"{100 * v / tot:5.1f}%  ?")
            continue
        f, ln = key
        if f not in src:
            p = [os.path.join(dp, f) for dp, _, fs in os.walk(os.path.dirname(os.path.abspath(obj)) + "/..") if f in fs]
            src[f] = open(p[0]).read().splitlines() if p else []
        text = src[f][ln - 1].strip() if ln - 1 < len(src[f]) else ""
        print(f"{100 * v / tot:5.1f}%  {f}:{ln:<5d} {text[:100]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 40)
