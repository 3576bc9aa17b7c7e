"""The attention backward's kernel variants give the same gradients (B200).

At head dim 64 the backward runs the two-stream kernels (bsattn_dkdv_ds / bsattn_dq_ds): each CTA deals its
units to two independent pipelines. The variant is chosen once per process from the environment, so every
variant runs in its own subprocess on the same seeded inputs:
  * default (units dealt by entry count), LX_ATTN_DS_DEAL=0 (units alternate between the streams): a unit's
    math does not depend on its stream, so dQ, dK and dV are bit-identical;
  * the entry-alternating ping-pong kernels (LX_ATTN_DKDV_DS=0 LX_ATTN_DQ_DS=0): dK / dV accumulate the same
    entries in the same order, so they are bit-identical; dQ differs only in the summation order of the bf16
    dS row sums of its common-mode correction.
The shape gives some CTAs more than the 64 units the two-stream kernels deal (the rest alternate)."""

import os
import subprocess
import sys
from pathlib import Path

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent

_CHILD = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
from paper_2510_15964_b200 import block_sparse as BS, patterns as PT
n_items, s, H, hd, ab = 24, 4096, 16, 64, 128
d = H * hd
g = torch.Generator().manual_seed(5)
qkv = (torch.randn(n_items * s, 3 * d, generator=g) * 0.5).to("cuda", torch.bfloat16)
dO = (torch.randn(n_items * s, d, generator=g) * 0.1).to("cuda", torch.bfloat16)
pool = PT.build_pool(s // ab)
dp = PT.device_pool(pool, torch.device("cuda"), s, ab)
names = list(pool)
rng = np.random.default_rng(7)
pidx = torch.tensor(rng.integers(0, len(names), size=(n_items, H)), dtype=torch.int32, device="cuda")
Q, K, V = qkv[:, :d], qkv[:, d:2 * d], qkv[:, 2 * d:]
o, lse = BS.attention_forward(Q, K, V, 3 * d, n_items, s, H, hd, pidx, H, dp, 0.125)
dqkv = torch.full_like(qkv, float("nan"))
BS.attention_backward(Q, K, V, o, dO, 3 * d, n_items, s, H, hd, pidx, H, dp, 0.125, lse,
                      dqkv[:, :d], dqkv[:, d:2 * d], dqkv[:, 2 * d:])
torch.cuda.synchronize()
torch.save(dqkv.cpu(), sys.argv[2])
"""


def _run(tmp_path, name: str, env: dict) -> torch.Tensor:
    out = tmp_path / f"{name}.pt"
    e = dict(os.environ, **env)
    r = subprocess.run([sys.executable, "-c", _CHILD, str(ROOT), str(out)], env=e, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return torch.load(out)


def test_two_stream_backward_variants(tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    dealt = _run(tmp_path, "dealt", {})
    alt = _run(tmp_path, "alternate", {"LX_ATTN_DS_DEAL": "0"})
    pp = _run(tmp_path, "pingpong", {"LX_ATTN_DKDV_DS": "0", "LX_ATTN_DQ_DS": "0"})
    d = dealt.shape[1] // 3
    assert torch.isfinite(dealt.float()).all()
    assert torch.equal(dealt, alt)
    assert torch.equal(dealt[:, d:], pp[:, d:])  # dK, dV
    dq, dq_pp = dealt[:, :d].float(), pp[:, :d].float()
    assert (dq - dq_pp).abs().max() <= 1e-2 * dq_pp.abs().max()
