#!/usr/bin/env python
"""Phase timeline (clock64 stamps, lx_debug_set_gemm_trace) of the two K1 scoring GEMMs at cfg3 shapes:
the attention-predictor projection (B*m = 184 rows x 8192 outputs, K = 2048 hi/lo) and the MLP mask GEMM
(4096 tokens x 512 blocks, K = 2048 hi/lo), cold L2. Stamps per CTA: 0 start, 1 end, 2 first stage landed (MMA),
3 last MMA issued, 4 epilogue got the accumulator, 5 epilogue done."""
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2510_15964_b200 import _abi  # noqa: E402

B, s, d, H, r, n_blk = 8, 512, 2048, 32, 128, 512
m = 23
dev = torch.device("cuda")
g = torch.Generator(device="cuda").manual_seed(0)
xs = torch.randn(B * m, d, device=dev, generator=g).to(torch.bfloat16)
wqk = (torch.randn(2 * H * r, 2 * d, device=dev, generator=g) * 0.05).to(torch.bfloat16)
proj = torch.empty(B * m, 2 * H * r, device=dev)
h = torch.randn(B * s, d, device=dev, generator=g).to(torch.bfloat16)
wa = (torch.randn(n_blk, 2 * d, device=dev, generator=g) * 0.05).to(torch.bfloat16)
bits = torch.zeros(B * (s // 32) * 16, dtype=torch.int32, device=dev)
counts = torch.zeros(B, dtype=torch.int32, device=dev)
ids = torch.zeros(B, n_blk, dtype=torch.int32, device=dev)
pos = torch.zeros(B, n_blk, dtype=torch.int32, device=dev)
pk = torch.zeros(8, dtype=torch.int32, device=dev)
pidx = torch.zeros(B, H, dtype=torch.int32, device=dev)
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
st = _abi.stream_handle()
buf = torch.zeros(160, 32, dtype=torch.int64, device=dev)


def attn():
    _abi.call("lx_predict_attention_patterns", xs.data_ptr(), B, m, d, wqk.data_ptr(), H, r, 2, 0.1, 0.9, 8, pk.data_ptr(),
              pk.data_ptr(), 1, 0, proj.data_ptr(), pidx.data_ptr(), None, st)


def mlp():
    _abi.call("lx_predict_mlp_mask", h.data_ptr(), B, s, d, wa.data_ptr(), n_blk, 2, 0.5, 0, bits.data_ptr(),
              counts.data_ptr(), ids.data_ptr(), pos.data_ptr(), None, st)


for name, fn in (("attn_pred", attn), ("mlp_mask", mlp)):
    ts = []
    for i in range(13):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        if i >= 3:
            ts.append(a.elapsed_time(b) * 1e3)
    flush.fill_(1)
    buf.zero_()
    _abi.call("lx_debug_set_gemm_trace", buf.data_ptr())
    fn()
    torch.cuda.synchronize()
    _abi.call("lx_debug_set_gemm_trace", None)
    t = buf.cpu().numpy().astype(np.int64)[:148]
    act = t[:, 2] > 0
    t0 = t[act, 0].min()
    rel = lambda k: (t[act, k] - t0)
    print(f"{name}: {statistics.median(ts):.1f} us (cold, whole call); CTAs with a tile {act.sum()}")
    for k, lab in ((0, "start"), (2, "first stage"), (3, "last MMA"), (4, "epi got acc"), (5, "epi done"), (1, "end")):
        v = rel(k)
        print(f"   {lab:12s} min {v.min():7d} med {int(np.median(v)):7d} max {v.max():7d} cyc")
