"""Per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) of each probed C-ABI call from an ncu
launch list of one step: {config: {abi name: bytes per call}} for bench.py's roofline `traffic` field.
python tools/traffic_db.py launches.csv cfg3 > profiles/r02_ncu_traffic.json"""
import collections
import csv
import json
import sys

# the kernels each probed C-ABI call launches (per call, in order)
CALLS = {
    "lx_neuron_fc1": ["gemm_sm100_kernel<3, 2, 512, 2, 1>"],
    "lx_neuron_fc2": ["gemm_sm100_kernel<4, 3, 256, 1, 1>"],
    "lx_neuron_fc2_dgrad": ["gemm_sm100_kernel<3, 4, 512, 2, 1>"],
    "lx_neuron_fc1_dgrad": ["gemm_sm100_kernel<4, 5, 256, 1, 1>"],
    "lx_bsattn_fwd_tc": ["bsattn_fwd_tc_kernel<64>"],
    "lx_bsattn_bwd_tc": ["bsattn_prep_kernel<64>", "bsattn_dkdv_ds_kernel<64>", "bsattn_dq_ds_kernel<64>"],
    "lx_predict_mlp_mask": ["gemm_sm100_kernel<6, 6, 256, 2, 1>", "mask_compact_kernel"],
    "lx_predict_attention_patterns": ["gemm_sm100_kernel<6, 0, 256, 2, 1>", "attn_pattern_kernel"],
}
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
hdr = rows[hi]
ci = {h: i for i, h in enumerate(hdr)}
per = collections.defaultdict(float)
names = {}
for r in rows[hi + 1:]:
    if len(r) < len(hdr) or not r[ci["Metric Name"]].startswith("dram__bytes"):
        continue
    u = r[ci["Metric Unit"]]
    per[r[ci["ID"]]] += float(r[ci["Metric Value"]].replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    names[r[ci["ID"]]] = r[ci["Kernel Name"]]
by_k = collections.defaultdict(list)
for lid, b in per.items():
    by_k[names[lid]].append(b)
out = {}
for call, ks in CALLS.items():
    tot = 0.0
    for k in ks:
        hits = [v for n, v in by_k.items() if k in n]
        if not hits or not hits[0]:
            tot = None
            break
        tot += sum(hits[0]) / len(hits[0])
    out[call] = round(tot) if tot is not None else None
print(json.dumps({sys.argv[2]: out, "source": "ncu launch list of one eager cfg3 step (tools/ncu_r2.sh), mean per call"}, indent=1))
