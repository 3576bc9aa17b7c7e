"""Summarise an ncu --set full report: key throughput metrics + the top stalled SASS lines.
python tools/ncu_hot.py report.ncu-rep [n_lines]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25


def page(kind, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", kind, "--csv", *extra], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


raw = page("raw")
h, v = raw[0], raw[2]
want = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_shared_mem", "sm__ctas_launched.sum", "launch__grid_size"]
for w in want:
    for i, name in enumerate(h):
        if name.endswith(w) or name == w:
            print(f"{name} = {v[i]}")
            break
src = page("source", ["--print-source", "sass"])
hdr = src[1]
rows = src[2:]
iS = hdr.index("Warp Stall Sampling (All Samples)")
tot = sum(int(r[iS]) for r in rows if len(r) > iS and r[iS].isdigit())
print(f"stall samples: {tot}")
for r in sorted((r for r in rows if len(r) > iS and r[iS].isdigit()), key=lambda r: -int(r[iS]))[:n]:
    print(f"{int(r[iS]):6d} {100 * int(r[iS]) / tot:5.1f}%  {r[0][-5:]}  {r[1].strip()[:100]}")
