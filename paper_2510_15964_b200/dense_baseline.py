"""Dense comparison step: the same model semantics (pre-LN, non-causal attention,
no positional embedding, tied head, LoRA on wq/wv/w1/w2, Adam) written as a plain
PyTorch bf16 module — cuBLAS GEMMs and F.scaled_dot_product_attention, autograd
backward. This is the "dense cuBLAS/SDPA bf16 step" the north star compares
against; it is a baseline, not part of the product path.

Hardened so the comparison is not against a soft target:
  * the LM head + cross-entropy is a chunked fused function (logits of a row chunk are
    recomputed in the backward, no [M, V] fp32 tensor is kept), as production PEFT stacks do;
  * the whole step (forward, backward, fused Adam) is captured once in a CUDA graph
    (`capture()` / `replay()`), so the baseline is not launch-bound either.
"""

from __future__ import annotations

import torch
import torch.nn.functional as F


class _ChunkedLmHeadCE(torch.autograd.Function):
    """mean CE(hf @ emb^T, tgt) over rows, computed per row chunk; backward recomputes each chunk's
    logits (bf16 GEMM, fp32 accumulate) instead of storing them."""

    @staticmethod
    def forward(ctx, hf, emb, tgt, chunk: int):
        M = hf.shape[0]
        lse = torch.empty(M, dtype=torch.float32, device=hf.device)
        tl = torch.empty(M, dtype=torch.float32, device=hf.device)
        for r0 in range(0, M, chunk):
            lg = torch.mm(hf[r0 : r0 + chunk], emb.t(), out_dtype=torch.float32)
            lse[r0 : r0 + chunk] = torch.logsumexp(lg, dim=1)
            tl[r0 : r0 + chunk] = lg.gather(1, tgt[r0 : r0 + chunk, None])[:, 0]
        ctx.save_for_backward(hf, emb, tgt, lse)
        ctx.chunk = chunk
        return (lse - tl).mean()

    @staticmethod
    def backward(ctx, g):
        hf, emb, tgt, lse = ctx.saved_tensors
        M, chunk = hf.shape[0], ctx.chunk
        d_hf = torch.empty_like(hf)
        for r0 in range(0, M, chunk):
            lg = torch.mm(hf[r0 : r0 + chunk], emb.t(), out_dtype=torch.float32)
            p = torch.exp(lg - lse[r0 : r0 + chunk, None])
            p.scatter_add_(1, tgt[r0 : r0 + chunk, None], torch.full_like(p[:, :1], -1.0))
            d_hf[r0 : r0 + chunk] = (p * (g / M)).to(hf.dtype) @ emb
        return d_hf, None, None, None


class DenseLoraStep:
    def __init__(self, model, lr: float = 1e-3, loss_chunk: int = 1024):
        """Shares the frozen bf16 weights of a paper_2510_15964_b200.model.Model."""
        self.m = model
        self.loss_chunk = loss_chunk
        self.params = []
        self.lora = {}
        for (i, t), ad in model.lora.items():
            a = ad.a.detach().clone().requires_grad_(True)
            b = ad.b.detach().clone().requires_grad_(True)
            self.lora[(i, t)] = (a, b, ad.scaling)
            self.params += [a, b]
        self.opt = torch.optim.Adam(self.params, lr=lr, betas=(0.9, 0.999), eps=1e-8, fused=True, capturable=True)
        self.graph = None

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
        return _ChunkedLmHeadCE.apply(hf.reshape(B * s, d), m.weights.emb, tgt.reshape(-1).contiguous(), self.loss_chunk)

    def step(self, tokens: torch.Tensor) -> torch.Tensor:
        self.opt.zero_grad(set_to_none=False)
        loss = self.loss(tokens)
        loss.backward()
        self.opt.step()
        return loss.detach()

    # CUDA graph of the whole step (forward, backward, fused capturable Adam)
    def capture(self, tokens: torch.Tensor, warmup: int = 3) -> None:
        self.static_tokens = tokens.clone()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            for _ in range(warmup):
                self.step(self.static_tokens)
        torch.cuda.current_stream().wait_stream(side)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self.static_loss = self.step(self.static_tokens)

    def replay(self, tokens: torch.Tensor | None = None) -> torch.Tensor:
        if tokens is not None:
            self.static_tokens.copy_(tokens, non_blocking=True)
        self.graph.replay()
        return self.static_loss
