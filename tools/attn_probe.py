"""One block-sparse attention fwd+bwd at cfg2 shapes (B 4, s 1024, H 32, hd 64) bracketed by
cudaProfilerStart/Stop, for ncu --profile-from-start off.  python tools/attn_probe.py [sparsity] [attn_blk]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench_ops import attn_layout  # noqa: E402
from oracle.sf_oracle import make_rng  # noqa: E402
from paper_2510_15964_b200 import block_sparse as BS, patterns as PT  # noqa: E402

sp = float(sys.argv[1]) if len(sys.argv) > 1 else 0.0
ab = int(sys.argv[2]) if len(sys.argv) > 2 else 64
B, s, H, hd = 4, 1024, 32, 64
d, M, n_b = H * hd, B * s, s // ab
rng = make_rng(7)
grids = np.zeros((H, n_b, n_b), bool)
for h in range(H):
    cs = np.asarray(attn_layout(n_b, sp, rng))
    grids[h, cs[:, 0], cs[:, 1]] = True
dp = PT.DevicePool([f"h{h}" for h in range(H)], None, None, None, s, ab)
dp.tables = torch.from_numpy(PT.tables_from_grids(grids, s, ab)).cuda()
dp.tables128 = torch.from_numpy(PT.tables128_from_grids(grids, s, ab)).cuda()
pidx = torch.arange(H, dtype=torch.int32, device="cuda")[None]
qkv = torch.randn(M, 3 * d, device="cuda").to(torch.bfloat16)
dO = (torch.randn(M, d, device="cuda") * 0.1).to(torch.bfloat16)
dqkv = torch.empty_like(qkv)
Q, K, V = qkv[:, :d], qkv[:, d:2 * d], qkv[:, 2 * d:]


def run():
    o, lse = BS.attention_forward(Q, K, V, 3 * d, B, s, H, hd, pidx, 0, dp, 1.0 / 8)
    BS.attention_backward(Q, K, V, o, dO, 3 * d, B, s, H, hd, pidx, 0, dp, 1.0 / 8, lse, dqkv[:, :d], dqkv[:, d:2 * d],
                          dqkv[:, 2 * d:])


for _ in range(3):
    run()
torch.cuda.synchronize()
torch.cuda.profiler.start()
run()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("done")
