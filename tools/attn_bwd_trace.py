"""Unit timeline of the persistent ping-pong dK/dV kernel (debug clock64 stamps) at cfg3 layer shapes.
Per CTA, for its first 5 units k: K/V landed (MMA view), first entry S ready, first entry dS stored, dK/dV
accumulated, drained. Usage: python tools/attn_bwd_trace.py [pattern=blockdiag]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2510_15964_b200 import _abi, block_sparse as BS, patterns as PT  # noqa: E402

B, s, H, hd, ab = 8, 512, 32, 64, 64
pat = sys.argv[1] if len(sys.argv) > 1 else "blockdiag"
d = H * hd
dev = torch.device("cuda")
qkv = (torch.randn(B * s, 3 * d, device=dev) * 0.5).to(torch.bfloat16)
dO = (torch.randn(B * s, d, device=dev) * 0.1).to(torch.bfloat16)
pool = PT.build_pool(s // ab)
dp = PT.device_pool(pool, dev, s, ab)
pidx = torch.full((B, H), list(pool).index(pat), dtype=torch.int32, device=dev)
Q, K, V = qkv[:, :d], qkv[:, d:2 * d], qkv[:, 2 * d:]
o, lse = BS.attention_forward(Q, K, V, 3 * d, B, s, H, hd, pidx, H, dp, 0.125)
dqkv = torch.empty_like(qkv)


def run():
    BS.attention_backward(Q, K, V, o, dO, 3 * d, B, s, H, hd, pidx, H, dp, 0.125, lse, dqkv[:, :d], dqkv[:, d:2 * d],
                          dqkv[:, 2 * d:])


for _ in range(3):
    run()
torch.cuda.synchronize()
buf = torch.zeros(4096, 32, dtype=torch.int64, device=dev)
_abi.call("lx_debug_set_attn_trace", buf.data_ptr())
run()
torch.cuda.synchronize()
_abi.call("lx_debug_set_attn_trace", None)
t = buf.cpu().numpy().astype(np.int64)[:148]
rel = t - t[:, 0:1]
names = ["K/V landed", "S(0) ready", "dS(0) stored", "acc done", "drained"]
for k in range(5):
    print(f"unit {k}: " + "  ".join(f"{names[i]} {np.median(rel[:, 2 + 5 * k + i]):7.0f}" for i in range(5)))
print("MMA: " + "  ".join(f"{nm} {np.median(rel[:, sl]):7.0f}" for nm, sl in (("u0 dV/dP", 27), ("u0 dK", 28), ("u1 dV/dP", 29), ("u1 dK", 30))))
