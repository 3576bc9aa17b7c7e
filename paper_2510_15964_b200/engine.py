"""Device-resident fine-tune step (the inner loop of sf/harness.py:396-427).

`FinetuneEngine.step(tokens)` runs predict -> forward -> loss -> backward ->
(all-reduce hook) -> Adam entirely on the GPU with no host synchronisation,
so the whole step can be captured once in a CUDA graph and replayed (the
launch-bound pattern the B200 playbook asks for). The LM head never
materialises the full [B*s, V] logits: cross-entropy and its gradient are
computed in row chunks (tied embedding, sf/model.py:449-472).
"""

from __future__ import annotations

import numpy as np
import torch

from . import autograd as AG, model as M


# LX_LMHEAD_FUSED=0: fp32 logits from cuBLAS + the CE kernel (the round-1 path) instead of the fused-epilogue logits
# GEMM (lx_lm_head_ce), for measurements
_LMHEAD_FUSED = __import__("os").environ.get("LX_LMHEAD_FUSED", "1") != "0"


def lm_head_loss_and_grad(hf: torch.Tensor, emb: torch.Tensor, targets: torch.Tensor, s: int, chunk: int = 4096):
    """Mean CE over positions (per-item mean, then batch mean) and d(sum of per-item losses)/d hf.
    hf bf16 [M, d]; emb bf16 [V, d]; targets int64 [M]. Returns (loss fp32 scalar tensor, d_hf fp32 [M, d]).
    Default: no fp32 logits exist -- the logits GEMM's epilogue keeps per-segment softmax statistics and stores
    bf16 exp(l - m_seg), a combine kernel forms the loss, a rescale pass turns that into the bf16 gradient
    (lx_lm_head_ce), and d_hf = g emb is one library GEMM."""
    from . import _abi

    Mr, V = hf.shape[0], emb.shape[0]
    if _LMHEAD_FUSED:
        dev = hf.device
        nseg = _abi.lib().lx_lm_head_ce_nseg(V)
        ldg = (V + 7) // 8 * 8
        d_hf = torch.empty(Mr, hf.shape[1], dtype=torch.float32, device=dev)
        row_loss = torch.empty(Mr, dtype=torch.float32, device=dev)
        tg = targets.contiguous()
        for r0 in range(0, Mr, chunk):
            r1 = min(Mr, r0 + chunk)
            g = torch.empty(r1 - r0, ldg, dtype=torch.bfloat16, device=dev)
            stats = torch.empty(r1 - r0, 2 * nseg, dtype=torch.float32, device=dev)
            coef = torch.empty(r1 - r0, nseg, dtype=torch.float32, device=dev)
            tl = torch.empty(r1 - r0, dtype=torch.float32, device=dev)
            _abi.call("lx_lm_head_ce", hf[r0:r1].data_ptr(), hf.stride(0), r1 - r0, hf.shape[1], emb.data_ptr(), V,
                      tg[r0:r1].data_ptr(), 1.0 / s, g.data_ptr(), ldg, stats.data_ptr(), coef.data_ptr(), tl.data_ptr(),
                      row_loss[r0:].data_ptr(), _abi.stream_handle(dev))
            d_hf[r0:r1] = M._mm_f32(g[:, :V], emb)
        return row_loss.mean(), d_hf
    d_hf = torch.empty(Mr, hf.shape[1], dtype=torch.float32, device=hf.device)
    row_loss = torch.empty(Mr, dtype=torch.float32, device=hf.device)
    tg = targets.contiguous()
    for r0 in range(0, Mr, chunk):
        r1 = min(Mr, r0 + chunk)
        lg = M._mm_f32(hf[r0:r1], emb.t())  # [c, V] fp32 (cuBLAS)
        gb = torch.empty(r1 - r0, V, dtype=torch.bfloat16, device=hf.device)
        _abi.call("lx_cross_entropy", lg.data_ptr(), r1 - r0, V, tg[r0:r1].data_ptr(), 1.0 / s, row_loss[r0:].data_ptr(),
                  gb.data_ptr(), _abi.stream_handle(hf.device))  # fused CE fwd+bwd, per-item mean (sf/model.py:472)
        d_hf[r0:r1] = M._mm_f32(gb, emb)
    return row_loss.mean(), d_hf


class FinetuneEngine:
    """Fused fine-tune step over a batch of B sequences of length s (tokens [B, s+1])."""

    def __init__(self, model: M.Model, state: M.PeftState, provider, lr: float, loss_chunk: int = 0, grad_hook=None,
                 grad_sync=None):
        """grad_hook(flat): one in-place reduction of the flat mean-gradient buffer after the step (dp.make_grad_hook);
        grad_sync: a dp.BucketedGradSync issuing that reduction per layer group during the backward instead."""
        self.model, self.state, self.provider, self.lr = model, state, provider, lr
        self.grad_sync = grad_sync
        import os

        # LM-head row chunk: 4096 rows (824 MB of fp32 logits at V = 50272) measured fastest at cfg3 (18.69 vs
        # 18.84 ms/step at 1024 rows, 18.94 at 512: the larger GEMMs win over L2 residency of the CE sweeps)
        self.loss_chunk = loss_chunk or int(os.environ.get("LX_LOSS_CHUNK", "4096"))
        self.grad_hook = grad_hook  # called with the flat mean-gradient buffer (e.g. NCCL all-reduce)
        self.flat_grad = torch.zeros_like(state.flat)
        self.graph = None
        self.static_tokens = None
        self.static_loss = None
        self._grad_views = {}
        self._layer_range = {}  # layer -> [lo, hi) of its trainables in the flat buffer (contiguous per layer)
        base = state.flat.data_ptr()
        for name, p in state.params.items():
            off = (p.data_ptr() - base) // 4
            self._grad_views[name] = self.flat_grad[off : off + p.numel()].view(p.shape)
            layer = int(name.split(".")[1])
            lo, hi = self._layer_range.get(layer, (off, off))
            self._layer_range[layer] = (min(lo, off), max(hi, off + p.numel()))
        self.last_masks = None
        M.ensure_lora_packs(model)  # packed LoRA operands, refreshed at the start of every step

    def _cg_stream(self):
        """Side stream for the LoRA / BitFit column reductions (LX_CG_SIDE_STREAM=0 keeps them inline)."""
        import os

        if os.environ.get("LX_CG_SIDE_STREAM", "1") == "0":
            return None
        if getattr(self, "_side", None) is None:
            self._side = torch.cuda.Stream(device=self.model.device)
        return self._side

    # -------------------------------------------------------------- one step (capturable)
    def _step(self, tokens: torch.Tensor) -> torch.Tensor:
        m = self.model
        B, s1 = tokens.shape
        s = s1 - 1
        inp, tgt = tokens[:, :-1], tokens[:, 1:].reshape(-1)
        M.refresh_lora_packs(m)  # one launch: LoRA factors (updated by Adam) -> bf16 packs / K-extended rows
        h = torch.nn.functional.embedding(inp, m.weights.emb).float()  # index_select gather, not advanced indexing
        caches = []
        for layer in range(m.dims.n_layers):
            h, c = M.block_forward(h, m, layer, self.provider)
            caches.append(c)
        hf, cf = M.layernorm_forward(h, m.weights.lnf_g, m.weights.lnf_b)
        loss, d_hf = lm_head_loss_and_grad(hf, m.weights.emb, tgt, s, self.loss_chunk)
        # gradient reductions write straight into the flat buffer, pre-scaled by 1/B (sf/harness.py:415)
        grads = AG.FlatGrads(self._grad_views, 1.0 / B)
        dh, dh_bf = AG.layernorm_backward(d_hf, cf, want_bf16=True)
        cg = None
        side = self._cg_stream()
        if side is not None:  # fork the side stream from this (possibly capturing) stream, so the join below is legal
            side.wait_stream(torch.cuda.current_stream())  # even when no column reduction runs on it (adapter)
        sync = self.grad_sync
        # buckets only where every trainable is written by the column reductions (LoRA, BitFit); the adapter's
        # torch-op gradients are copied in at the end and reduced by finish()
        bucketed = sync is not None and m.peft_method != "adapter"
        if sync is not None:
            sync.begin()
        group = []
        for k, layer in enumerate(reversed(range(m.dims.n_layers))):
            cg = cg or AG._CgBatch(grads, B, s, stream=side)
            dh, dh_bf = AG.block_backward(dh, m, layer, caches[layer], None, grads, dh_bf, inplace=True, cg=cg)
            group.append(layer)
            if k % AG.CG_LAYERS == AG.CG_LAYERS - 1:  # CG_LAYERS layers' column reductions per group launch
                cg.flush()
                cg = None
                if bucketed:
                    self._bucket(group, side)
                group = []
        if cg is not None:
            cg.flush()
            if bucketed:
                self._bucket(group, side)
        if side is not None:
            torch.cuda.current_stream().wait_stream(side)  # join: Adam reads every gradient
        self.last_masks = [c["masks"] for c in caches]
        for name, view in self._grad_views.items():
            t = grads.get(name)
            if t is None:
                view.zero_()  # unreached trainables get zero gradients (sf/autograd.py:191-194)
            elif t is not view:
                view.copy_(t).mul_(1.0 / B)  # gradients produced by torch ops (adapter path)
        if sync is not None:
            sync.finish(self.flat_grad)  # the rest, then the compute stream waits for the collectives
        return loss

    def _bucket(self, layers, producer_stream) -> None:
        rs = [self._layer_range[i] for i in layers if i in self._layer_range]
        if rs:
            self.grad_sync.bucket(self.flat_grad, min(r[0] for r in rs), max(r[1] for r in rs), producer_stream)

    def _finish(self) -> None:
        """Data-parallel gradient reduction hook (unless bucketed inside the step), then Adam (float64 moments,
        sf/autograd.py:203-225)."""
        if self.grad_hook is not None and self.grad_sync is None:
            self.grad_hook(self.flat_grad)
        self.state.step += 1
        from . import _abi

        st = self.state
        _abi.call("lx_adam_step", st.flat.data_ptr(), self.flat_grad.data_ptr(), st.m.data_ptr(), st.v.data_ptr(),
                  st.flat.numel(), float(self.lr), 0.9, 0.999, 1e-8, st.step, _abi.stream_handle(st.flat.device))

    def step(self, tokens) -> torch.Tensor:
        """Eager step (tokens host or device). Returns the loss as a device scalar."""
        tok = torch.as_tensor(np.asarray(tokens) if not torch.is_tensor(tokens) else tokens)
        tok = tok.to(self.model.device, torch.int64, non_blocking=True)
        loss = self._step(tok)
        self._finish()
        return loss

    # -------------------------------------------------------------- CUDA graph
    def capture(self, example_tokens: torch.Tensor, warmup: int = 2) -> None:
        """Capture forward+backward+grad-reduction (not Adam, whose bias correction depends on
        the step count) into one CUDA graph; Adam runs as a handful of elementwise kernels."""
        self.static_tokens = example_tokens.to(self.model.device, torch.int64).clone()
        torch.cuda.empty_cache()  # eager steps' cached blocks back to the driver: the graph pool is separate
        if hasattr(self.provider, "timing"):
            self.provider.timing = False  # no timing events inside a graph
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            for _ in range(warmup):
                self._step(self.static_tokens)
        torch.cuda.current_stream().wait_stream(side)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self.static_loss = self._step(self.static_tokens)

    def replay(self, tokens=None) -> torch.Tensor:
        if tokens is not None:
            self.static_tokens.copy_(tokens, non_blocking=True)
        self.graph.replay()
        self._finish()
        return self.static_loss
