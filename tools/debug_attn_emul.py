"""Diagnostics: device attention (fwd + bwd) vs the bf16 rounding-point emulation (oracle/bf16_emul.py) for one
(item, head) at cfg1-like shapes, with a common mode in q/k like the model's."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import bf16_emul as E, sf_oracle as O  # noqa: E402
from paper_2510_15964_b200 import block_sparse as BS, patterns as PT  # noqa: E402


def rel(a, b):
    a = np.asarray(a.detach().float().cpu() if torch.is_tensor(a) else a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


dev = torch.device("cuda")
for s, ab, cm, dens in ((256, 16, 0.0, 1.0), (256, 16, 3.0, 1.0), (256, 16, 3.0, 0.3), (256, 64, 3.0, 0.5), (512, 64, 3.0, 1.0)):
    rng = np.random.default_rng(s + ab)
    hd, H = 64, 1
    n_b = s // ab
    q, k, v, do = (rng.standard_normal((s, hd)).astype(np.float32) for _ in range(4))
    c = rng.standard_normal(hd).astype(np.float32) * cm
    q, k = q + c, k + c
    do *= 0.01
    grid = rng.random((n_b, n_b)) < dens
    np.fill_diagonal(grid, True)
    e = E.Emul()
    qb, kb, vb, dob = (E.bf16(a) for a in (q, k, v, do))
    coords = np.argwhere(grid)
    oe, lse_e, mask = E.attention_forward_dev(e, qb, kb, vb, coords, ab, 0.125)
    dqe, dke, dve = E.attention_backward_dev(e, qb, kb, vb, oe, dob, lse_e, mask, 0.125)
    dp = PT.DevicePool(["x"], None, None, torch.from_numpy(PT.tables128_from_grids(grid[None], s, ab)).to(dev), s, ab)
    pidx = torch.zeros(1, 1, dtype=torch.int32, device=dev)
    qkv = torch.from_numpy(np.concatenate([qb, kb, vb], 1)).to(dev, torch.bfloat16)
    d = H * hd
    Q, K, V = qkv[:, :d], qkv[:, d:2 * d], qkv[:, 2 * d:]
    o, lse = BS.attention_forward(Q, K, V, 3 * d, 1, s, H, hd, pidx, 0, dp, 0.125)
    dqkv = torch.empty_like(qkv)
    BS.attention_backward(Q, K, V, o, torch.from_numpy(dob).to(dev, torch.bfloat16), 3 * d, 1, s, H, hd, pidx, 0, dp, 0.125, lse,
                          dqkv[:, :d], dqkv[:, d:2 * d], dqkv[:, 2 * d:])
    torch.cuda.synchronize()
    f = O.dense_masked_attention(qb, kb, vb, coords, ab, 0.125)
    print(f"s {s} ab {ab} common {cm} density {dens}: o {rel(o, oe):.2e} (vs f64 {rel(o, f):.2e}) lse {np.abs(lse.cpu().numpy()[0,0]-lse_e).max():.2e} "
          f"dq {rel(dqkv[:, :d], dqe):.2e} dk {rel(dqkv[:, d:2*d], dke):.2e} dv {rel(dqkv[:, 2*d:], dve):.2e}")
