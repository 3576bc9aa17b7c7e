"""Time lx_cross_entropy alone on one LM-head chunk (1024 x 50272 fp32 logits, cfg3) with CUDA events.
LX_CE_CTAS_PER_SM selects the persistent grid (read once per process)."""
import json
import os

import torch

from paper_2510_15964_b200 import _abi

rows, V, reps = int(os.environ.get("ROWS", "1024")), 50272, 50
dev = torch.device("cuda:0")
logits = torch.randn(rows, V, device=dev)
tgt = torch.randint(0, V, (rows,), device=dev)
row_loss = torch.empty(rows, device=dev)
gb = torch.empty(rows, V, dtype=torch.bfloat16, device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
h = _abi.stream_handle(dev)
ts = []
for i in range(reps + 5):
    flush.zero_()
    logits.add_(0.0)  # logits freshly written (as by the GEMM), part of them L2-resident
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    _abi.call("lx_cross_entropy", logits.data_ptr(), rows, V, tgt.data_ptr(), 1.0 / 512, row_loss.data_ptr(), gb.data_ptr(), h)
    b.record()
    torch.cuda.synchronize()
    if i >= 5:
        ts.append(a.elapsed_time(b) * 1e3)
ts.sort()
alg = rows * V * (4 + 2)  # one fp32 read + one bf16 write per logit
print(json.dumps({"ctas_per_sm": os.environ.get("LX_CE_CTAS_PER_SM", "default"), "rows": rows, "us_median": ts[len(ts) // 2],
                  "us_min": ts[0], "alg_GBps": alg / (ts[len(ts) // 2] * 1e-6) / 1e9}))
