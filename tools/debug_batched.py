"""Diagnostics: the batched-items fixture (tests/test_gpu_model.py) run as one batch of 3 and item by item
on the device, against the bf16 rounding-point oracle; intermediate activations compared per layer."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import bf16_emul as E, sf_oracle as O  # noqa: E402
from paper_2510_15964_b200 import autograd as AG, model as M  # noqa: E402


def rel(a, b):
    a = np.asarray(a.detach().float().cpu() if torch.is_tensor(a) else a, np.float64)
    b = np.asarray(b.detach().float().cpu() if torch.is_tensor(b) else b, np.float64)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


dev = torch.device("cuda")
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
print("patterns", pat)
masks = [M.LayerMasks([pat[b][i] for b in range(B)], nms[:, i]) for i in range(dims.n_layers)]
logits, cache = M.model_forward(m, toks[:, :-1], masks)
grads = AG.model_backward(m, cache, M.loss_backward(logits, toks[:, 1:]), masks)
per_item = []
for b in range(B):
    mb = [M.LayerMasks(pat[b][i], nms[b, i]) for i in range(dims.n_layers)]
    lg1, c1 = M.model_forward(m, toks[b, :-1], mb)
    g1 = AG.model_backward(m, c1, M.loss_backward(lg1, toks[b, 1:]), mb)
    per_item.append((lg1, c1, g1))
    om_masks = [(pat[b][i], nms[b, i]) for i in range(dims.n_layers)]
    e = E.Emul()
    lge, ce = E.model_forward(e, om, toks[b, :-1], om_masks)
    ge = E.model_backward(e, om, ce, O.loss_backward(lge, toks[b, 1:]))
    s = dims.seq_len
    print(f"item {b}: logits batch-vs-single {rel(logits[b], lg1):.2e}  single-vs-emul {rel(lg1, lge):.2e}")
    for i in range(dims.n_layers):
        cb, cs, cemu = cache["blocks"][i], c1["blocks"][i], ce["blocks"][i]
        qkv_b = cb["attn"]["qkv"][b * s:(b + 1) * s]
        q_e = np.concatenate([cemu["attn"]["q"], cemu["attn"]["k"], cemu["attn"]["v"]], 1)
        o_b = cb["attn"]["o"][b * s:(b + 1) * s]
        a_b = cb["mlp"]["a"].values[b * s:(b + 1) * s]
        na = cemu["mlp"]["a"].shape[1]
        print(f"  layer {i}: qkv b-vs-emul {rel(qkv_b, q_e):.2e} o b-vs-emul {rel(o_b, cemu['attn']['heads']):.2e} "
              f"o single-vs-emul {rel(cs['attn']['o'], cemu['attn']['heads']):.2e} "
              f"a b-vs-emul {rel(a_b[:, :na], cemu['mlp']['a']):.2e} a single-vs-emul {rel(cs['mlp']['a'].values[:, :na], cemu['mlp']['a']):.2e}")
    for n in ge:
        if np.abs(ge[n]).max() > 0:
            print(f"   {n:30s} single-vs-emul {rel(g1[n], ge[n]):.3e}")
gsum = {n: sum(pi[2][n] for pi in per_item) for n in grads}
for n in grads:
    if float(gsum[n].abs().max()) > 0:
        print(f"   {n:30s} batch-vs-sum-of-singles {rel(grads[n], gsum[n]):.3e}")
