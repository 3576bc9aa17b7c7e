"""Per-CTA balance of the two-stream attention backward kernels in one eager cfg3 step (debug clock64 stamps).

The trace buffer keeps the last launch of each kernel (layer 0's backward). Per CTA and stream: cycles from
CTA start to the stream's last drain, units and entries. Usage: python tools/attn_ds_trace.py
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2510_15964_b200 import _abi  # noqa: E402
from paper_2510_15964_b200.engine import FinetuneEngine  # noqa: E402

cfg = bench.CONFIGS["cfg3"]
dev = torch.device("cuda", 0)
model, state, prov = bench.build_workload(cfg, dev, 0, 0.85, 0.75, peft="lora")
eng = FinetuneEngine(model, state, prov, lr=1e-4)
tok = torch.randint(0, cfg["V"], (cfg["B"], cfg["s"] + 1), device=dev)
for _ in range(3):
    eng.step(tok)
torch.cuda.synchronize()
buf = torch.zeros(4096, 32, dtype=torch.int64, device=dev)
_abi.call("lx_debug_set_attn_trace", buf.data_ptr())
eng.step(tok)
torch.cuda.synchronize()
_abi.call("lx_debug_set_attn_trace", None)
t = buf.cpu().numpy().astype(np.int64)
n_cta = min(148, int((t[:, 0] != 0).sum()))
t = t[:n_cta]
for name, b in (("dK/dV", 0), ("dQ", 8)):
    end = np.stack([t[:, b + 1] - t[:, b], t[:, b + 2] - t[:, b]], 1)
    units = np.stack([t[:, b + 3] >> 32, t[:, b + 4] >> 32], 1)
    ents = np.stack([t[:, b + 3] & 0xFFFFFFFF, t[:, b + 4] & 0xFFFFFFFF], 1)
    cta = end.max(1)
    print(f"{name}: {n_cta} CTAs; CTA cycles median {np.median(cta):.0f} max {cta.max()} min {cta.min()}; "
          f"entries per CTA median {np.median(ents.sum(1)):.0f} max {ents.sum(1).max()} min {ents.sum(1).min()}; "
          f"units per CTA {np.median(units.sum(1)):.0f}; cycles per entry (per CTA) {np.median(cta / np.maximum(ents.sum(1), 1)):.0f}")
    print(f"  stream imbalance |end0-end1| median {np.median(np.abs(end[:, 0] - end[:, 1])):.0f}; "
          f"corr(entries, cycles) {np.corrcoef(ents.sum(1), cta)[0, 1]:.2f}")
    hist = np.bincount(ents.sum(1))
    print("  entries/CTA histogram:", {i: int(c) for i, c in enumerate(hist) if c})
    order = np.argsort(cta)
    for i in list(order[:3]) + list(order[-3:]):
        print(f"  cta {i}: cycles {end[i].tolist()} units {units[i].tolist()} entries {ents[i].tolist()}")
t = t[:148]
print(f"unit dealing (after the PDL wait): dK/dV {np.median(t[:, 0] - t[:, 6]):.0f} dQ {np.median(t[:, 8] - t[:, 7]):.0f} cycles")
