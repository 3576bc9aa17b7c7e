"""TEST INFRASTRUCTURE ONLY — generate the offline-pipeline fixtures from the UNMODIFIED
reference: a `.tnsc` file written by sf/containers.py:save_tensors (tests/golden/ref_container.tnsc),
and predictor training runs of sf/predictor.py (train_attn_predictor, train_mlp_predictor,
mlp_truth_labels, init_*), all in tests/golden/offline.npz.

    python oracle/make_golden_offline.py
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"


def main() -> None:
    sys.path.insert(0, str(REF))
    from sparseft import containers as C, predictor as P  # noqa: E402

    rng = np.random.default_rng(77)
    g = {}
    # ---- container written by the reference
    ct = {
        "w.f32": rng.standard_normal((3, 5)).astype(np.float32),
        "w.f64": rng.standard_normal((2, 3, 4)),
        "ids": rng.integers(-5, 1 << 40, size=7).astype(np.int64),
        "colmaj": np.asfortranarray(rng.standard_normal((4, 6)).astype(np.float32)),
        "scalar": np.array(3.25),
        "empty": np.zeros((0, 3), np.float32),
    }
    C.save_tensors(OUT / "ref_container.tnsc", ct, column_major={"colmaj"})
    for k, v in ct.items():
        g[f"ct/{k}"] = np.array(v, order="C")
    g["ct/names"] = np.array(list(ct))
    # ---- attention predictor training (noise 0: deterministic), plus one noisy run's loss
    d, H, r, s, n = 32, 2, 4, 64, 3
    idx = P.downsample_indices(s)
    xs = [rng.standard_normal((s, d)).astype(np.float32) for _ in range(n)]
    raws = []
    for i in range(n):
        per = []
        for h in range(H):
            a = rng.standard_normal((s, 6)).astype(np.float32)
            per.append((a @ a.T).astype(np.float64) * 0.3)
        raws.append(per)
    for tag, noise in (("a0", 0.0), ("a1", 0.05)):
        params = P.init_attn_predictor(d, H, rank=r, seed=5)
        g[f"{tag}/wq0"], g[f"{tag}/wk0"] = np.stack(params.wq_hat), np.stack(params.wk_hat)
        cfg = P.PredictorTrainConfig(noise_std=noise, epochs=25, lr=1e-2)
        loss = P.train_attn_predictor(xs, raws, params, cfg, seed=9)
        g[f"{tag}/wq"], g[f"{tag}/wk"] = np.stack(params.wq_hat), np.stack(params.wk_hat)
        g[f"{tag}/loss"] = np.array(loss)
        g[f"{tag}/meta"] = np.array([d, H, r, s, n, noise, 25, 1e-2])
    for i in range(n):
        g[f"a/x{i}"] = xs[i][idx]
        for h in range(H):
            g[f"a/raw{i}.{h}"] = raws[i][h][np.ix_(idx, idx)]
    # ---- MLP predictor training and truth labels
    d, s, d_ff, blk, n = 32, 40, 100, 16, 2
    n_blk = -(-d_ff // blk)
    xm = [rng.standard_normal((s, d)).astype(np.float32) for _ in range(n)]
    zs = [(rng.standard_normal((s, d_ff)) - 1.6).astype(np.float32) for _ in range(n)]
    for tag, noise in (("m0", 0.0), ("m1", 0.05)):
        params = P.init_mlp_predictor(d, n_blk, seed=6)
        g[f"{tag}/wa0"] = params.wa_hat.copy()
        cfg = P.PredictorTrainConfig(noise_std=noise, epochs=25, lr=1e-2, recall_weight=4.0)
        loss = P.train_mlp_predictor(xm, zs, blk, params, cfg, seed=11)
        g[f"{tag}/wa"] = params.wa_hat
        g[f"{tag}/loss"] = np.array(loss)
    g["m/meta"] = np.array([d, s, d_ff, blk, n])
    for i in range(n):
        g[f"m/x{i}"], g[f"m/z{i}"] = xm[i], zs[i]
        g[f"m/labels{i}"] = P.mlp_truth_labels(zs[i], blk)
    # ragged label case (d_ff not a multiple of blk, blk > 32)
    z = (rng.standard_normal((9, 130)) - 2.0).astype(np.float32)
    g["lab/z"], g["lab/blk"], g["lab/labels"] = z, np.array(40), P.mlp_truth_labels(z, 40)
    # ---- init draws
    ap = P.init_attn_predictor(48, 3, rank=None, seed=12)
    g["init/wq"], g["init/wk"] = np.stack(ap.wq_hat), np.stack(ap.wk_hat)
    g["init/wa"] = P.init_mlp_predictor(48, 5, seed=13).wa_hat
    np.savez_compressed(OUT / "offline.npz", **g)
    print("wrote", OUT / "offline.npz", OUT / "ref_container.tnsc")


if __name__ == "__main__":
    main()
