"""Summarise an ncu launch list (`--metrics gpu__time_duration.sum[,dram__bytes_read.sum,dram__bytes_write.sum] --csv`)
by kernel: launches, serialised time, DRAM bytes per launch and the achieved DRAM rate."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
hdr = rows[hi]
ci = {h: i for i, h in enumerate(hdr)}
per = collections.defaultdict(dict)  # launch id -> metrics
names = {}
for r in rows[hi + 1:]:
    if len(r) < len(hdr):
        continue
    lid = r[ci["ID"]]
    v = float(r[ci["Metric Value"]].replace(",", ""))
    u = r[ci["Metric Unit"]]
    m = r[ci["Metric Name"]]
    if m == "gpu__time_duration.sum":
        v = v / 1e3 if u in ("nsecond", "ns") else v * 1e3 if u in ("msecond", "ms") else v  # -> us
    else:
        v = v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    per[lid][m] = v
    names[lid] = r[ci["Kernel Name"]].split("(")[0][:100]
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
tot = 0.0
for lid, mm in per.items():
    t = mm.get("gpu__time_duration.sum", 0.0)
    b = mm.get("dram__bytes_read.sum", 0.0) + mm.get("dram__bytes_write.sum", 0.0)
    a = agg[names[lid]]
    a[0] += 1
    a[1] += t
    a[2] += b
    tot += t
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
print(f"total {tot / 1e3:.2f} ms over {len(per)} launches (ncu-serialised, cold caches)")
print(f"{'ms':>8} {'share':>6} {'n':>5} {'us/launch':>10} {'MB/launch':>10} {'GB/s':>7}  kernel")
for k, (n, t, b) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
    print(f"{t / 1e3:8.3f} {100 * t / tot:5.1f}% {n:5d} {t / n:10.1f} {b / n / 1e6:10.2f} {b / max(t, 1e-9) / 1e3:7.0f}  {k}")
