"""Phase timeline of the tcgen05 attention dK/dV kernel at cfg3 layer shapes (debug stamps, clock64).
Per CTA: 0 start, 1 K/V landed, per q-tile e<4: 2+6e q/dO landed (S MMA issue), 3+6e S in TMEM,
4+6e P stored, 5+6e dP in TMEM, 6+6e dS stored; 26 last dK MMA done; 27 epilogue end."""
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
n_cta = (s // 128) * H * B
buf = torch.zeros(n_cta, 32, dtype=torch.int64, device=dev)
_abi.call("lx_debug_set_attn_trace", buf.data_ptr())
run()
torch.cuda.synchronize()
_abi.call("lx_debug_set_attn_trace", None)
t = buf.cpu().numpy().astype(np.int64)  # the dq kernel runs last and overwrites slots it stamps; dkdv slots are its own
t0 = t[:, 0:1]
rel = t - t0
print(f"CTA lifetime (0 -> 27) mean {np.mean(t[:, 27] - t[:, 0]):.0f} cycles")
print(f"start -> K/V landed {np.mean(rel[:, 1]):.0f}")
for e in range(4):
    b = 2 + 6 * e
    print(f"e={e}: qdO {np.mean(rel[:, b]):7.0f}  S {np.mean(rel[:, b+1]):7.0f}  P {np.mean(rel[:, b+2]):7.0f}  "
          f"dP {np.mean(rel[:, b+3]):7.0f}  dS {np.mean(rel[:, b+4]):7.0f}")
print(f"dK done {np.mean(rel[:, 26]):.0f}  epi end {np.mean(rel[:, 27]):.0f}")
sm = t[:, 31]
span = [t[sm == i, 27].max() - t[sm == i, 0].min() for i in np.unique(sm)]
print(f"per-SM busy span mean {np.mean(span):.0f} cycles over {len(span)} SMs; CTAs per SM {n_cta / len(span):.1f}")
