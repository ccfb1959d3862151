"""Key metrics from `ncu -i X.ncu-rep --page raw --csv` exports (X.raw.csv), for profiles/."""
import csv
import sys

sys.path.insert(0, __file__.rsplit("/", 1)[0])
from ncu_summary import KEYS  # noqa: E402


def main(path):
    rows = list(csv.reader(open(path)))
    rows = [r for r in rows if r and not r[0].startswith("==")]
    h, units = rows[0], rows[1]
    ki = h.index("Kernel Name")
    print(f"# {path}")
    for row in rows[2:]:
        print(f"## {row[ki][:150]}")
        for k in KEYS:
            if k in h:
                i = h.index(k)
                print(f"  {k:62s} {row[i]:>16s} {units[i]}")
        st = []
        for i, n in enumerate(h):
            if n.startswith("smsp__pcsamp_warps_issue_stalled") and not n.endswith("not_issued"):
                try:
                    st.append((float(row[i].replace(",", "")), n.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(v for v, _ in st) or 1.0
        print("  stalls: " + ", ".join(f"{n} {100 * v / tot:.0f}%" for v, n in sorted(st, reverse=True)[:6]))
        print()


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
