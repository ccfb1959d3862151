"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per-kernel totals and shares."""
import collections
import csv
import re
import sys


def summarise(path, top=30):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows[hi + 1:]:
        v = float(r[vi].replace(",", ""))
        v = {"ns": v / 1e3, "us": v, "usecond": v, "nsecond": v / 1e3, "ms": v * 1e3, "msecond": v * 1e3}.get(r[ui], v)
        name = re.split(r"\((bk::|long|const|int,|double)", r[ki])[0].strip()
        tot[name] += v
        cnt[name] += 1
    T = sum(tot.values())
    out = [f"# {path}: {sum(cnt.values())} launches, {T:.1f} us total (ncu: cold-cache, serialised)",
           f"{'total_us':>10} {'share':>6} {'n':>5} {'avg_us':>8}  kernel"]
    for n, v in sorted(tot.items(), key=lambda x: -x[1])[:top]:
        out.append(f"{v:10.1f} {100 * v / T:5.1f}% {cnt[n]:5d} {v / cnt[n]:8.2f}  {n}")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarise(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30))
