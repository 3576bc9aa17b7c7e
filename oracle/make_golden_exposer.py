"""TEST INFRASTRUCTURE ONLY — generate tests/golden/exposer.npz from the UNMODIFIED
reference: the exposer oracle mode (sf/exposer.py:47-111) through the reference's own
OracleProvider / ShadowyProvider (sf/harness.py:157-190), driven with minimal duck-typed
model objects carrying exactly the fields those methods read.

Run in the build container (the reference does not exist on the GPU box):

    python oracle/make_golden_exposer.py
"""

from __future__ import annotations

import sys
from pathlib import Path
from types import SimpleNamespace as NS

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"


def main() -> None:
    sys.path.insert(0, str(REF))
    from sparseft import exposer as E, harness as HN, patterns as PT  # noqa: E402

    rng = np.random.default_rng(20251015)
    g = {}
    # ---- attention: exact probabilities -> block masses -> per-head / shadowy patterns
    cases = [(32, 2, 32, 2), (64, 4, 64, 4), (64, 8, 32, 2), (96, 4, 64, 2), (128, 8, 64, 4), (128, 4, 128, 2),
             (256, 8, 64, 2), (64, 2, 16, 1)]
    for c, (s, n_b, d, H) in enumerate(cases):
        tau = float([0.5, 0.8, 0.95, 0.99][c % 4])
        pos = np.arange(s)[:, None] / s
        feats = np.concatenate([np.sin(pos * np.arange(1, d // 2 + 1) * 3.0), np.cos(pos * np.arange(1, d // 2 + 1) * 3.0)], 1)
        x = (feats * (1.0 + c % 3) + 0.3 * rng.standard_normal((s, d))).astype(np.float32)
        sharp = [0.05, 0.3, 1.0][c % 3]
        wq = (rng.standard_normal((d, d)) * sharp).astype(np.float32)
        wk = wq.copy() if c % 2 else (rng.standard_normal((d, d)) * sharp).astype(np.float32)
        bq = (0.1 * rng.standard_normal(d)).astype(np.float32)
        bk = (0.1 * rng.standard_normal(d)).astype(np.float32)
        lw = NS(wq=wq, bq=bq, wk=wk, bk=bk)
        dims = NS(head_dim=d // H, n_heads=H, n_b=n_b)
        pool = PT.build_pool(n_b)
        model = NS(weights=NS(layers=[lw]), dims=dims, pool=pool)
        probs, _ = E.exact_attention(x, lw, dims)
        g[f"att{c}/x"] = x
        g[f"att{c}/wq"], g[f"att{c}/bq"], g[f"att{c}/wk"], g[f"att{c}/bk"] = wq, bq, wk, bk
        g[f"att{c}/meta"] = np.array([s, n_b, d, H, tau])
        g[f"att{c}/mass"] = np.stack([E.block_mass(p, n_b) for p in probs])
        g[f"att{c}/pids"] = np.array(HN.OracleProvider(model, 0.0, tau)._attn(0, x))
        g[f"att{c}/shadowy"] = np.array(HN.ShadowyProvider(model, tau)._attn(0, x))
    g["n_att"] = np.array(len(cases))
    # ---- MLP: z = h W1 + b1 (+ s (h A) B) -> block importance -> theta filter
    mcases = [(16, 32, 64, 16, 0.0, 4), (40, 64, 256, 16, 0.1, 8), (7, 32, 100, 16, 0.5, 0), (64, 64, 512, 32, 0.3, 4),
              (1, 16, 48, 4, 1.0, 0), (33, 48, 96, 1, 0.2, 2)]
    for c, (s, d, d_ff, blk, theta, r) in enumerate(mcases):
        h = rng.standard_normal((s, d)).astype(np.float32)
        w1 = (rng.standard_normal((d, d_ff)) * 0.2).astype(np.float32)
        b1 = (rng.standard_normal(d_ff) * 0.1 - 0.3).astype(np.float32)
        lora = {}
        if r:
            a = (rng.standard_normal((d, r)) * 0.1).astype(np.float32)
            b = (rng.standard_normal((r, d_ff)) * 0.1).astype(np.float32)
            scaling = 2.0
            lora[(0, "w1")] = NS(a=a, b=b, scaling=scaling)
            g[f"mlp{c}/a"], g[f"mlp{c}/b"] = a, b
        model = NS(weights=NS(layers=[NS(mlp=NS(w1=w1), b1=b1)]), lora=lora, dims=NS(blk_size=blk))
        g[f"mlp{c}/h"], g[f"mlp{c}/w1"], g[f"mlp{c}/b1"] = h, w1, b1
        g[f"mlp{c}/meta"] = np.array([s, d, d_ff, blk, theta, r, 2.0])
        g[f"mlp{c}/mask"] = HN.OracleProvider(model, theta, 0.95)._mlp(0, h)
    g["n_mlp"] = np.array(len(mcases))
    OUT.mkdir(parents=True, exist_ok=True)
    np.savez_compressed(OUT / "exposer.npz", **g)
    print("wrote", OUT / "exposer.npz", sum(v.nbytes for v in g.values()), "bytes")


if __name__ == "__main__":
    main()
