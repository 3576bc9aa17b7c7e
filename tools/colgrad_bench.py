"""Isolated lx_colgrad_group timing at the cfg3 sublayer groups (attention: dB_q, dB_v, dA_q, dA_v;
MLP: dB2, dA2[cols], dB1[:,cols], dA1). CUDA events, inputs resident, L2 flushed between reps.

    python tools/colgrad_bench.py [reps]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2510_15964_b200 import neuron_ops as N  # noqa: E402

dev = torch.device("cuda", 0)
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
B, s, d, f, r, blk = 8, 512, 2048, 8192, 8, 16
M = B * s
g = torch.Generator(device=dev).manual_seed(0)
h1 = torch.randn(M, d, device=dev, generator=g).to(torch.bfloat16)
dqkv = torch.randn(M, 3 * d, device=dev, generator=g).to(torch.bfloat16)
ax = torch.randn(M, 16, device=dev, generator=g)
dax = torch.randn(M, 16, device=dev, generator=g)
# MLP: ~11% of blocks active, the same blocks in every item (as the injected predictor sparsity)
n_blk = f // blk
act = torch.zeros(B, n_blk, dtype=torch.bool, device=dev)
act[:, torch.randperm(n_blk, generator=torch.Generator().manual_seed(1))[: int(0.113 * n_blk)].to(dev)] = True
nm = N.lower_mask(act, n_blk, blk, B, dev)
fa = int(nm.counts.max()) * blk
a = torch.randn(M, fa, device=dev, generator=g).to(torch.bfloat16)
dz = torch.randn(M, fa, device=dev, generator=g).to(torch.bfloat16)
dO = torch.randn(M, d, device=dev, generator=g).to(torch.bfloat16)
h2 = torch.randn(M, d, device=dev, generator=g).to(torch.bfloat16)
ax2, dax2, ax1, dax1 = (torch.randn(M, r, device=dev, generator=g) for _ in range(4))
G = [torch.empty(r, f, device=dev) for _ in range(8)]
attn = [N.colgrad_problem(ax[:, :8], dqkv[:, :d], d, r, 1.0, G[0], d, 1),
        N.colgrad_problem(ax[:, 8:], dqkv[:, 2 * d:], d, r, 1.0, G[1], d, 1),
        N.colgrad_problem(dax[:, :8], h1, d, r, 1.0, G[2], 1, r),
        N.colgrad_problem(dax[:, 8:], h1, d, r, 1.0, G[3], 1, r)]
mlp = [N.colgrad_problem(ax2, dO, d, r, 1.0, G[4], d, 1),
       N.colgrad_problem(dax2, a, f, r, 1.0, G[5], 1, r, masks=nm, blk=blk),
       N.colgrad_problem(ax1, dz, f, r, 1.0, G[6], f, 1, masks=nm, blk=blk),
       N.colgrad_problem(dax1, h2, d, r, 1.0, G[7], 1, r)]
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for name, probs, nbytes in [("attn", attn, (4 * M * d) * 2), ("mlp", mlp, (2 * M * d + 2 * M * fa) * 2)]:
    for single in (False, True):
        for _ in range(3):
            N.colgrad_group(probs, B, s)
        ts = []
        for _ in range(reps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            if single:
                for p in probs:
                    N.colgrad_group([p], B, s)
            else:
                N.colgrad_group(probs, B, s)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        ts.sort()
        us = ts[len(ts) // 2]
        print(f"{name:5s} {'per-problem' if single else 'grouped':11s} {us:8.1f} us  {nbytes / us / 1e3:7.0f} GB/s (algorithmic bytes {nbytes / 1e6:.1f} MB)")
