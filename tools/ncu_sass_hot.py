"""Summarise an ncu report: key metrics + hottest SASS lines (stall samples).
    python tools/ncu_sass_hot.py report.ncu-rep [n_hot]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
nhot = int(sys.argv[2]) if len(sys.argv) > 2 else 25
if rep.endswith(".ncu-rep"):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
else:   # prefix of tools/ncu_cap.sh CSV exports
    raw = open(rep + ".raw.csv").read()
    src = open(rep + ".sass.csv").read()
r = list(csv.reader(io.StringIO(raw)))
h, u, v = r[0], r[1], r[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]
for name, unit, val in zip(h, u, v):
    if name in want or ("pcsamp_warps_issue_stalled" in name and "not_issued" not in name):
        try:
            if float(val.replace(",", "")) == 0:
                continue
        except ValueError:
            pass
        print(f"{name:70s} {unit:10s} {val}")
rows = list(csv.reader(io.StringIO(src)))
hh = rows[1]
iS = hh.index("Warp Stall Sampling (All Samples)")
iE = hh.index("Instructions Executed")
data = rows[2:]
tot = sum(float(x[iS] or 0) for x in data)
print("total samples", tot)
for x in sorted(data, key=lambda x: -float(x[iS] or 0))[:nhot]:
    print(x[0][-5:], x[iS], x[iE], x[1][:100])
