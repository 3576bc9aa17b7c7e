"""Summarise an ncu --set full report: duration, DRAM traffic, pipe utilisation + the top stalled SASS lines.
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
h, u, v = raw[0], raw[1], raw[2]
print(f"kernel: {v[h.index('Kernel Name')][:160]}")
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "lts__t_bytes.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_shared_mem", "launch__grid_size", "launch__block_size",
        "sm__cycles_elapsed.avg.per_second"]
for w in want:
    for i, name in enumerate(h):
        if name == w or name.endswith("." + w):
            print(f"  {w} = {v[i]} {u[i]}")
            break
src = page("source", ["--print-source", "sass"])
if len(src) > 2:
    hdr = src[1] if "Warp Stall Sampling (All Samples)" in src[1] else src[0]
    rows = src[2:]
    iS = hdr.index("Warp Stall Sampling (All Samples)")
    tot = sum(int(r[iS]) for r in rows if len(r) > iS and r[iS].isdigit())
    print(f"  stall samples: {tot}")
    for r in sorted((r for r in rows if len(r) > iS and r[iS].isdigit()), key=lambda r: -int(r[iS]))[:n]:
        print(f"  {int(r[iS]):6d} {100 * int(r[iS]) / max(tot, 1):5.1f}%  {r[0][-5:]}  {r[1].strip()[:100]}")
