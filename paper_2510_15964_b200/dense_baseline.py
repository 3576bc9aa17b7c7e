"""Dense comparison step: the same model semantics (pre-LN, non-causal attention,
no positional embedding, tied head, LoRA on wq/wv/w1/w2, Adam) written as a plain
PyTorch bf16 module — cuBLAS GEMMs and F.scaled_dot_product_attention, autograd
backward. This is the "dense cuBLAS/SDPA bf16 step" the north star compares
against; it is a baseline, not part of the product path."""

from __future__ import annotations

import torch
import torch.nn.functional as F


class DenseLoraStep:
    def __init__(self, model, lr: float = 1e-3):
        """Shares the frozen bf16 weights of a paper_2510_15964_b200.model.Model."""
        self.m = model
        self.params = []
        self.lora = {}
        for (i, t), ad in model.lora.items():
            a = ad.a.detach().clone().requires_grad_(True)
            b = ad.b.detach().clone().requires_grad_(True)
            self.lora[(i, t)] = (a, b, ad.scaling)
            self.params += [a, b]
        self.opt = torch.optim.Adam(self.params, lr=lr, betas=(0.9, 0.999), eps=1e-8, fused=True)

    def _lin(self, x, w, b, key):
        y = x @ w
        if b is not None:
            y = y + b.to(y.dtype)
        if key in self.lora:
            a, bb, s = self.lora[key]
            y = y + s * ((x @ a.to(x.dtype)) @ bb.to(x.dtype))
        return y

    def loss(self, tokens: torch.Tensor) -> torch.Tensor:
        m = self.m
        dims = m.dims
        d, H, hd = dims.d_model, dims.n_heads, dims.head_dim
        inp, tgt = tokens[:, :-1], tokens[:, 1:]
        B, s = inp.shape
        h = torch.nn.functional.embedding(inp, m.weights.emb)
        for i, lw in enumerate(m.weights.layers):
            x = F.layer_norm(h.float(), (d,), lw.ln1_g, lw.ln1_b, 1e-5).to(torch.bfloat16)
            q = self._lin(x, lw.wq, lw.bq, (i, "wq"))
            k = self._lin(x, lw.wk, lw.bk, (i, "wk"))
            v = self._lin(x, lw.wv, lw.bv, (i, "wv"))
            q, k, v = (t.view(B, s, H, hd).transpose(1, 2) for t in (q, k, v))
            o = F.scaled_dot_product_attention(q, k, v, is_causal=False).transpose(1, 2).reshape(B, s, d)
            h = h + self._lin(o, lw.wo, lw.bo, (i, "wo")).float()
            x = F.layer_norm(h, (d,), lw.ln2_g, lw.ln2_b, 1e-5).to(torch.bfloat16)
            z = torch.relu(self._lin(x, lw.mlp.w1_t.t(), lw.b1, (i, "w1")))
            h = h + self._lin(z, lw.mlp.w2, lw.b2, (i, "w2")).float()
        hf = F.layer_norm(h, (d,), m.weights.lnf_g, m.weights.lnf_b, 1e-5).to(torch.bfloat16)
        logits = hf @ m.weights.emb.t()
        return F.cross_entropy(logits.view(-1, logits.shape[-1]).float(), tgt.reshape(-1))

    def step(self, tokens: torch.Tensor) -> torch.Tensor:
        self.opt.zero_grad(set_to_none=True)
        loss = self.loss(tokens)
        loss.backward()
        self.opt.step()
        return loss.detach()
