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
    import tests.test_gpu_model as TG

    e = E.Emul(relu=TG.device_relu(cache))
    lge, ce = E.model_forward(e, om, toks[:-1], masks_o)
    ge = E.model_backward(e, om, ce, O.loss_backward(lge, toks[1:]))
    print(f"== {peft}: logits dev-vs-fp32 {rel(lg, g[peft + '/logits']):.2e} dev-vs-emul {rel(lg, lge):.2e}")
    for n in ge:
        ref = g[f"{peft}/grad/{n}"]
        if np.abs(ref).max() == 0:
            continue
        print(f"   {n:36s} dev-emul {rel(gr[n], ge[n]):.3e}   dev-fp32 {rel(gr[n], ref):.3e}   emul-fp32 {rel(ge[n], ref):.3e}")

# the batched-items fixture of tests/test_gpu_model.py::test_batched_items_equal_per_item_loop
dims = O.Dims(128, 2, 256, 128, 2, 80, 16, 32)
om = O.build_model(dims, seed=11, peft="lora")
rng = np.random.default_rng(0)
for ad in om.lora.values():
    ad["b"] += (rng.standard_normal(ad["b"].shape) * 0.02).astype(np.float32)
mdims = M.ModelDims(dims.d_model, dims.n_heads, dims.d_ff, dims.seq_len, dims.n_layers, dims.vocab, dims.blk_size,
                    dims.attn_blk)
m = M.from_arrays(mdims, "lora", om.emb, om.layers, om.lnf_g, om.lnf_b, lora=om.lora, lora_targets=om.lora_targets,
                  device=dev)
B = 3
toks = rng.integers(0, dims.vocab, size=(B, dims.seq_len + 1))
pids = list(om.pool)
pat = [[[pids[rng.integers(len(pids))] for _ in range(dims.n_heads)] for _ in range(dims.n_layers)] for _ in range(B)]
nms = rng.random((B, dims.n_layers, dims.n_blk)) < 0.5
masks = [M.LayerMasks([pat[b][i] for b in range(B)], nms[:, i]) for i in range(dims.n_layers)]
logits, cache = M.model_forward(m, toks[:, :-1], masks)
grads = AG.model_backward(m, cache, M.loss_backward(logits, toks[:, 1:]), masks)
ge, gf = {}, {}
for b in range(B):
    om_masks = [(pat[b][i], nms[b, i]) for i in range(dims.n_layers)]
    e = E.Emul(relu=TG.device_relu(cache, b))
    lge, ce = E.model_forward(e, om, toks[b, :-1], om_masks)
    for n, v in E.model_backward(e, om, ce, O.loss_backward(lge, toks[b, 1:])).items():
        ge[n] = ge.get(n, 0) + v
    lg, c = O.model_forward(om, toks[b, :-1], om_masks)
    for n, v in O.model_backward(om, c, O.loss_backward(lg, toks[b, 1:])).items():
        gf[n] = gf.get(n, 0) + v
    print(f"== batched item {b}: logits dev-emul {rel(logits[b], lge):.2e}, dev-fp32 {rel(logits[b], lg):.2e}")
for n in ge:
    if np.abs(gf[n]).max() > 0:
        print(f"   {n:36s} dev-emul {rel(grads[n], ge[n]):.3e}   dev-fp32 {rel(grads[n], gf[n]):.3e}   emul-fp32 {rel(ge[n], gf[n]):.3e}")
