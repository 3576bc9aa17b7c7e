"""Attention at cfg3 layer shapes (B 8, s 512, H 32, hd 64, attn_blk 64) with bench.py's pattern mix:
`n_local` heads blockdiag, the rest dense (or every head PATTERN). Times forward and backward (CUDA events,
median of 20) and reports credited FLOP/s (reference MAC convention) plus gathered MMA tiles.
    python tools/attn_bench.py [n_local=24] [pattern]       (ncu: --profile-from-start off; one profiled call each)"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2510_15964_b200 import block_sparse as BS, patterns as PT  # noqa: E402
from paper_2510_15964_b200.model import dp_nnz  # noqa: E402

B, s, H, hd, ab = 8, 512, 32, 64, 64
n_local = int(sys.argv[1]) if len(sys.argv) > 1 else 24
only = sys.argv[2] if len(sys.argv) > 2 else None
d = H * hd
dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(0)
qkv = (torch.randn(B * s, 3 * d, device=dev, generator=g) * 0.5).to(torch.bfloat16)
dO = (torch.randn(B * s, d, device=dev, generator=g) * 0.1).to(torch.bfloat16)
pool = PT.build_pool(s // ab)
dp = PT.device_pool(pool, dev, s, ab)
ids = list(pool)
row = [ids.index(only)] * H if only else [ids.index("blockdiag")] * n_local + [ids.index("dense")] * (H - n_local)
pidx = torch.tensor([row] * B, dtype=torch.int32, device=dev)
nnz = sum(dp_nnz(dp, i) for i in row) * B
Q, K, V = qkv[:, :d], qkv[:, d:2 * d], qkv[:, 2 * d:]
st = {}


def fwd():
    st["o"], st["lse"] = BS.attention_forward(Q, K, V, 3 * d, B, s, H, hd, pidx, H, dp, 0.125)


fwd()
dqkv = torch.empty_like(qkv)


def bwd():
    BS.attention_backward(Q, K, V, st["o"], dO, 3 * d, B, s, H, hd, pidx, H, dp, 0.125, st["lse"], dqkv[:, :d],
                          dqkv[:, d:2 * d], dqkv[:, 2 * d:])


def timeit(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


tab = dp.tables.cpu().numpy()
tiles = [PT.tables128_work(tab, i) for i in row]
for name, fn, mult in (("fwd", fwd, 4), ("bwd", bwd, 8)):
    ms = timeit(fn)
    fl = mult * nnz * ab * ab * hd
    print(f"{name}: {ms * 1e3:.1f} us, credited {fl / ms / 1e9:.1f} TFLOP/s, block density {nnz / (B * H * (s // ab) ** 2):.3f}, "
          f"gathered tiles fwd/dq {B * sum(t[0] for t in tiles)} dkdv {B * sum(t[1] for t in tiles)} of {B * H * (s // 128) ** 2}")
torch.cuda.cudart().cudaProfilerStart()
fwd()
bwd()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
