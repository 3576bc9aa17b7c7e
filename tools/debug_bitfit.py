"""Diagnostics: BitFit on the reference fixture, device vs the bf16 rounding-point oracle, MLP backward taps."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import bf16_emul as E, sf_oracle as O  # noqa: E402
from paper_2510_15964_b200 import autograd as AG, model as M  # noqa: E402


def rel(a, b):
    a = np.asarray(a.detach().float().cpu() if torch.is_tensor(a) else a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


g = dict(np.load(Path(__file__).resolve().parents[1] / "tests/golden/model.npz"))
dev = torch.device("cuda")
peft = "bitfit"
d, H, f, s, L, V, blk, ablk = (int(v) for v in g["dims"])
om = O.build_model(O.Dims(d, H, f, s, L, V, blk, ablk), seed=7, peft=peft)
for n, p in O.trainable_params(om).items():
    p[...] = g[f"{peft}/param/{n}"]
masks_o = [(list(g[f"{peft}/masks/{i}/heads"]), g[f"{peft}/masks/{i}/neuron"]) for i in range(L)]
m = M.from_arrays(M.ModelDims(d, H, f, s, L, V, blk, ablk), peft, om.emb, om.layers, om.lnf_g, om.lnf_b, device=dev)
toks = g[f"{peft}/tokens"]
AG.DEBUG_TAPS = {}
lg, cache = M.model_forward(m, toks[:-1], [M.LayerMasks(*x) for x in masks_o])
gr = AG.model_backward(m, cache, M.loss_backward(lg, toks[1:]), [M.LayerMasks(*x) for x in masks_o])
e = E.Emul()
lge, ce = E.model_forward(e, om, toks[:-1], masks_o)
ge = E.model_backward(e, om, ce, O.loss_backward(lge, toks[1:]))
for i in range(L):
    cm = ce["blocks"][i]["mlp"]
    na = cm["a"].shape[1]
    a_dev = cache["blocks"][i]["mlp"]["a"].values[:, :na].float().cpu().numpy()
    dz_dev = AG.DEBUG_TAPS[f"layers.{i}.dz"][:, :na].float().cpu().numpy()
    do_dev = AG.DEBUG_TAPS[f"layers.{i}.dO"].float().cpu().numpy()
    print(f"layer {i}: a {rel(a_dev, cm['a']):.2e} (relu flips {int(((a_dev > 0) != (cm['a'] > 0)).sum())}), dO {rel(do_dev, cm['dO']):.2e}, "
          f"dz {rel(dz_dev, cm['dz']):.2e}, dz ulp-diffs {int((dz_dev != cm['dz']).sum())} of {dz_dev.size}")
    colsum_dev = dz_dev.astype(np.float64).sum(0)
    colsum_em = cm["dz"].astype(np.float64).sum(0)
    gb = gr[f"layers.{i}.b1"].cpu().numpy()
    cols = cm["cols"]
    print(f"   b1 dev-vs-emul {rel(gb, ge[f'layers.{i}.b1']):.2e}; host colsum(dev dz) vs emul {rel(colsum_dev, colsum_em):.2e}; "
          f"dev b1 vs host colsum(dev dz) {rel(gb[cols], colsum_dev):.2e}; max|b1| {np.abs(colsum_em).max():.3e} max|dz| {np.abs(cm['dz']).max():.3e}")
