import csv, sys
for p in sys.argv[1:]:
    rows = list(csv.reader(open(p)))
    h, units, v = rows[0], rows[1], rows[2]
    d = dict(zip(h, v))
    print("==", p, d.get("Kernel Name")[:60], d.get("Grid Size"), d.get("Block Size"))
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sectors.avg.pct_of_peak_sustained_elapsed",
            "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_active",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
            "lts__t_bytes.sum", "l1tex__t_bytes.sum"]
    for k in keys:
        for hh in h:
            if hh.endswith(k) or hh == k:
                print(f"  {hh[-60:]:60s} {d[hh]} {units[h.index(hh)]}")
                break
    st = [(float(d[x].replace(',', '')), x) for x in h if "smsp__pcsamp_warps_issue_stalled_" in x and d[x] not in ("", "n/a") and not x.endswith("_not_issued")]
    st.sort(reverse=True)
    tot = sum(a for a, _ in st) or 1
    print("  stalls:", ", ".join(f"{x.split('stalled_')[-1]} {100*a/tot:.0f}%" for a, x in st[:6]))
