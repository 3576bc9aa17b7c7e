"""Phase timeline of the persistent ping-pong dK/dV kernel at cfg3 layer shapes (debug stamps, clock64).
Per CTA (its first unit): 0 start, 1 K/V landed; per q-tile e<4 (WG e%2): 2+4e S ready, 3+4e P stored,
4+4e dP ready, 5+4e dS stored; 18 dK/dV done, 19 unit epilogue done; 20 second unit done."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2510_15964_b200 import _abi, block_sparse as BS, patterns as PT  # noqa: E402

B, s, H, hd, ab = 8, 512, 32, 64, 64
d = H * hd
dev = torch.device("cuda")
qkv = (torch.randn(B * s, 3 * d, device=dev) * 0.5).to(torch.bfloat16)
dO = (torch.randn(B * s, d, device=dev) * 0.1).to(torch.bfloat16)
pool = PT.build_pool(s // ab)
dp = PT.device_pool(pool, dev, s, ab)
pidx = torch.full((B, H), list(pool).index("dense"), dtype=torch.int32, device=dev)
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
print(f"start -> K/V landed {np.mean(rel[:, 1]):.0f}")
for e in range(4):
    b = 2 + 4 * e
    print(f"e={e} (WG{e % 2}): S {np.mean(rel[:, b]):7.0f}  P {np.mean(rel[:, b + 1]):7.0f}  dP {np.mean(rel[:, b + 2]):7.0f}  "
          f"dS {np.mean(rel[:, b + 3]):7.0f}")
print(f"unit0 dK/dV done {np.mean(rel[:, 18]):.0f}  epilogue done {np.mean(rel[:, 19]):.0f}  unit1 done {np.mean(rel[:, 20]):.0f}")
