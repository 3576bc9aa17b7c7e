#!/usr/bin/env python
"""Predictor projection GEMM probe (cfg3: x_small [B*m = 184, 2048] x [Wq_hat|Wk_hat]^T [8192, 2048]):
device time of lx_gemm_bf16_tn alone and of the whole attention-pattern prediction, L2 flushed."""
import json, statistics, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2510_15964_b200 import _abi, patterns as PT, predictor as P

B, s, d, H, r, n_b = 8, 512, 2048, 32, 128, 8
m = len(P.downsample_indices(s))
g = torch.Generator(device="cuda").manual_seed(0)
xs = torch.randn(B * m, d, device="cuda", generator=g).to(torch.bfloat16)
w = torch.randn(2 * H * r, d, device="cuda", generator=g).to(torch.bfloat16) * 0.05
out = torch.empty(B * m, 2 * H * r, device="cuda")
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
params = P.AttnPredictorParams([torch.zeros(d, r)] * H, [torch.zeros(d, r)] * H)
params._dev[P._dev_key(torch.device("cuda"))] = w
pool = PT.build_pool(n_b)
def t(fn, reps=30, cold=True):
    for _ in range(3): fn()
    ts = []
    for _ in range(reps):
        if cold:
            flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); b.synchronize(); ts.append(a.elapsed_time(b) * 1e3)
    return statistics.median(ts)
st = _abi.stream_handle()
gemm = lambda: _abi.call("lx_gemm_bf16_tn", xs.data_ptr(), d, w.data_ptr(), d, out.data_ptr(), 2 * H * r, 1, B * m, 2 * H * r, d, 0, st)
full = lambda: P.attn_pattern_idx(xs, B, m, params, pool, n_b, P.PredictorTrainConfig())
ref = xs.float() @ w.float().t()
gemm(); torch.cuda.synchronize()
err = float((out - ref).abs().max() / ref.abs().max())
print(json.dumps({"gemm_us": round(t(gemm), 2), "gemm_warm_us": round(t(gemm, cold=False), 2), "predict_attn_us": round(t(full), 2), "rel_err": err,
                  "weights_mb": round(w.numel() * 2 / 2**20, 1)}))
