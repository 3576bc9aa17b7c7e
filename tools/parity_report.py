"""Per-tensor parity report on the reference's model fixture: device vs bf16 rounding-point oracle vs
float32 oracle, for LoRA / Adapter / BitFit (all tensors, no early stop). GPU only; diagnostics."""
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
for peft in ("lora", "adapter", "bitfit"):
    d, H, f, s, L, V, blk, ablk = (int(v) for v in g["dims"])
    om = O.build_model(O.Dims(d, H, f, s, L, V, blk, ablk), seed=7, peft=peft)
    for n, p in O.trainable_params(om).items():
        p[...] = g[f"{peft}/param/{n}"]
    masks_o = [(list(g[f"{peft}/masks/{i}/heads"]), g[f"{peft}/masks/{i}/neuron"]) for i in range(L)]
    dims = M.ModelDims(d, H, f, s, L, V, blk, ablk)
    m = M.from_arrays(dims, peft, om.emb, om.layers, om.lnf_g, om.lnf_b, lora=om.lora, adapters=om.adapters,
                      lora_targets=om.lora_targets, device=dev)
    toks = g[f"{peft}/tokens"]
    lg, cache = M.model_forward(m, toks[:-1], [M.LayerMasks(*x) for x in masks_o])
    gr = AG.model_backward(m, cache, M.loss_backward(lg, toks[1:]), [M.LayerMasks(*x) for x in masks_o])
    e = E.Emul()
    lge, ce = E.model_forward(e, om, toks[:-1], masks_o)
    ge = E.model_backward(e, om, ce, O.loss_backward(lge, toks[1:]))
    print(f"== {peft}: logits dev-vs-fp32 {rel(lg, g[peft + '/logits']):.2e} dev-vs-emul {rel(lg, lge):.2e}")
    for n in ge:
        ref = g[f"{peft}/grad/{n}"]
        if np.abs(ref).max() == 0:
            continue
        print(f"   {n:36s} dev-emul {rel(gr[n], ge[n]):.3e}   dev-fp32 {rel(gr[n], ref):.3e}   emul-fp32 {rel(ge[n], ref):.3e}")
