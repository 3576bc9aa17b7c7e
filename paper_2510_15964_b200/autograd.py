"""Hand-written backward for the trainable set only (drop-in for sf/autograd.py).

Inactive neuron blocks and attention blocks are never touched: the MLP
input-grad runs the tcgen05 gather-GEMMs over the forward's index lists, the
LoRA / BitFit gradients are deterministic skinny reductions over the packed
active columns (inactive rows/columns stay exactly 0, sf/autograd.py:89-90),
attention gradients flow through the block-sparse backward kernels only. The
dense projection input-grads are plain library GEMMs (model.proj_t); the q/k/v LoRA term
rides in the same GEMM by K-extension ([dqkv | dAx] x [W_qkv^T ; A^T]). Gradients are sums over the batch items (the
reference harness sums per-item gradients and divides by the batch size,
sf/harness.py:413-415).

The residual-stream gradient travels as (fp32, bf16) pairs: the LayerNorm
backward kernel accumulates in fp32 and emits the bf16 copy the next GEMMs
consume, so no separate conversion pass exists.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _abi
from . import model as M
from .block_sparse import attention_backward
from .errors import GradientError
from .neuron_ops import (ROWPROJ_SEG_MAX_K, colgrad_group, colgrad_problem, pack_active_rows2, rowproj, rowproj_packed,
                         rowproj_packed_seg)


def check_gradient_set(grads: dict, model: M.Model) -> None:
    """sf/autograd.py:28-38."""
    trainable = M.trainable_params(model)
    if set(grads) != set(trainable):
        missing = set(trainable) - set(grads)
        extra = set(grads) - set(trainable)
        raise GradientError(f"gradient set mismatch: missing={sorted(missing)}, extra={sorted(extra)}")
    for name, g in grads.items():
        if tuple(g.shape) != tuple(trainable[name].shape):
            raise GradientError(f"{name}: gradient shape {tuple(g.shape)} != param shape {tuple(trainable[name].shape)}")
    bad = [n for n, g in grads.items() if not bool(torch.isfinite(g).all())]
    if bad:
        raise GradientError(f"{bad[0]}: non-finite gradient")


def _acc(grads: dict, name: str, value: torch.Tensor) -> None:
    if name in grads:
        grads[name] = grads[name] + value
    else:
        grads[name] = value


class FlatGrads(dict):
    """Gradient sink of the step engine: a gradient whose name has a view in the flat gradient
    buffer is written there directly by its reduction kernel, pre-scaled (1/B for the batch mean),
    instead of being allocated and copied."""

    def __init__(self, views: dict, scale: float):
        super().__init__()
        self.views, self.scale = views, scale


# diagnostics and teacher-forced tests: when a dict, block_backward records its fp32 d_out under "<prefix>d_out"
# and mlp_backward its bf16 dO and dz under "<prefix>dO" / "<prefix>dz"
DEBUG_TAPS: dict | None = None

CG_LAYERS = 2  # layers whose LoRA / BitFit column reductions share one lx_colgrad_group launch (4: no gain)


class _CgBatch:
    """The LoRA / BitFit column reductions of one sublayer's backward, collected and run as one
    deterministic lx_colgrad_group launch. A gradient with a view in a FlatGrads buffer is written
    there directly (pre-scaled by the batch mean); others are accumulated after the launch."""

    def __init__(self, grads: dict, n_items: int, s: int, stream=None):
        self.grads, self.n_items, self.s = grads, n_items, s
        self.probs, self.post = [], []
        self.stream = stream  # side stream: the launch overlaps the following layers' backward

    def add(self, name, shape, p, x2, ncols, r, scale, g_sq, g_sc, masks=None, blk=1) -> None:
        g = self.grads
        if isinstance(g, FlatGrads) and name in g.views and name not in g:
            out = g.views[name]
            scale = scale * g.scale
            dict.__setitem__(g, name, out)
        else:
            out = torch.empty(shape, dtype=torch.float32, device=x2.device)
            self.post.append((name, out))
        self.probs.append(colgrad_problem(p, x2, ncols, r, scale, out, g_sq, g_sc, masks=masks, blk=blk))

    def flush(self) -> None:
        if self.probs and self.stream is not None and not self.post:
            # nothing downstream of the backward reads these gradients before the optimizer step, so the
            # group runs on a side stream (joined by the caller) and fills SMs the next layers leave idle
            main = torch.cuda.current_stream()
            self.stream.wait_stream(main)
            for pr in self.probs:
                for t in (pr["p"], pr["x"], pr["out"]):
                    if t is not None:
                        t.record_stream(self.stream)
                if pr["masks"] is not None:
                    pr["masks"].pos.record_stream(self.stream)
            with torch.cuda.stream(self.stream):
                colgrad_group(self.probs, self.n_items, self.s)
        elif self.probs:
            colgrad_group(self.probs, self.n_items, self.s)
        for name, out in self.post:
            _acc(self.grads, name, out)
        self.probs, self.post = [], []


def _bf16(t: torch.Tensor) -> torch.Tensor:
    return t if t.dtype == torch.bfloat16 else t.to(torch.bfloat16)


def lora_linear_backward(dz, w, adapter, cache, grads: dict, prefix: str, bias_name):
    """sf/autograd.py:48-58 (reference-API helper; the model uses the fused paths below).
    dz fp32 [M, d_out], w bf16 [d_in, d_out]. Returns dx fp32."""
    dx = M._mm_f32(dz.to(torch.bfloat16), w.t())
    if adapter is not None:
        d_ax = (dz @ adapter.b.t()) * adapter.scaling
        _acc(grads, f"{prefix}.lora_a", cache["x"].float().t() @ d_ax)
        _acc(grads, f"{prefix}.lora_b", adapter.scaling * (cache["ax"].t() @ dz))
        dx.addmm_(d_ax, adapter.a.t())
    if bias_name is not None:
        _acc(grads, bias_name, dz.sum(0))
    return dx


def layernorm_backward(dy, cache, accumulate_into: torch.Tensor | None = None, want_bf16: bool = False):
    """sf/autograd.py:61-66 on the fused kernel: returns (accumulate_into or 0) + LN'(dy) in fp32,
    and with want_bf16 also its bf16 copy (written by the same kernel)."""
    x = cache["x"]
    Mr, d = x.shape
    out = accumulate_into if accumulate_into is not None else torch.zeros(Mr, d, dtype=torch.float32, device=x.device)
    ob = torch.empty(Mr, d, dtype=torch.bfloat16, device=x.device) if want_bf16 else None
    dy2 = dy.reshape(Mr, d)
    if dy2.stride(1) != 1 or dy2.stride(0) != d:
        dy2 = dy2.contiguous()
    _abi.call("lx_layernorm_bwd", dy2.data_ptr(), int(dy2.dtype == torch.float32), x.data_ptr(), cache["gamma"].data_ptr(),
              cache["mean"].data_ptr(), cache["inv_std"].data_ptr(), Mr, d, out.data_ptr(), _abi.ptr(ob),
              _abi.stream_handle(x.device))
    return (out, ob) if want_bf16 else out


def adapter_backward(dy, ad: M.AdapterLayer, cache, grads: dict, prefix: str):
    """sf/autograd.py:69-75 on the fp32 adapter kernels (csrc/adapter.cu): one row pass (dh, dx) and one
    deterministic column reduction for the four gradients. Returns dx fp32."""
    dy = dy.float().reshape(-1, ad.w_up.shape[1]).contiguous()
    M, d = dy.shape
    r = ad.w_down.shape[1]
    dev = dy.device
    dh = torch.empty(M, r, dtype=torch.float32, device=dev)
    dx = torch.empty_like(dy)
    ws = torch.empty(int(_abi.lib().lx_adapter_ws_floats(d, r)), dtype=torch.float32, device=dev)
    g = {k: torch.empty_like(getattr(ad, k)) for k in ("w_down", "b_down", "w_up", "b_up")}
    x = cache["x"]
    _abi.call("lx_adapter_bwd", dy.data_ptr(), d, x.data_ptr(), x.stride(0), M, d, r, cache["z"].data_ptr(),
              ad.w_down.data_ptr(), ad.w_up.data_ptr(), dh.data_ptr(), dx.data_ptr(), d, ws.data_ptr(), 1.0,
              g["w_down"].data_ptr(), g["b_down"].data_ptr(), g["w_up"].data_ptr(), g["b_up"].data_ptr(),
              _abi.stream_handle(dev))
    for k, v in g.items():
        _acc(grads, f"{prefix}.{k}", v)
    return dx


def mlp_backward(d_out, cache, lw: M.LayerWeights, lora: dict, neuron_mask, dims: M.ModelDims, grads: dict,
                 prefix: str = "", bitfit: bool = False, cg: "_CgBatch | None" = None):
    """Backward of mlp_forward (sf/autograd.py:78-124). d_out [M, d] (bf16 preferred) -> dx bf16 [M, d]."""
    nm = cache["mask"]
    if neuron_mask is not None and neuron_mask is not nm:
        other = M.lower_mask(neuron_mask, nm.n_blk, nm.blk, nm.n_items, nm.pos.device)
        if not torch.equal(other.pos, nm.pos):
            raise GradientError("cache was produced with a different neuron mask")
    B, s = cache["n_items"], cache["s"]
    d, f, blk = dims.d_model, dims.d_ff, dims.blk_size
    x2, hid = cache["x"], cache["a"]
    a = hid.values
    dev = a.device
    dO = _bf16(d_out.reshape(-1, d)).contiguous()
    st = _abi.stream_handle(dev)
    own = cg is None  # a caller-provided batch (block_backward) is flushed by the caller
    cg = _CgBatch(grads, B, s) if own else cg
    if bitfit:
        cg.add(f"{prefix}b2", (d,), None, dO, d, 1, 1.0, 0, 1)
    ad1, ad2 = lora.get("w1"), lora.get("w2")
    lp = lw.lora_pack or {}
    dax2 = None
    if ad2 is not None:
        r2 = ad2.rank
        if lp.get("b2") is not None:
            dax2 = rowproj_packed(dO, B, s, d, lp["b2"], r2, scale=ad2.scaling)  # dO B2^T * s
        else:
            dax2 = rowproj(dO, B, s, d, ad2.b, 1, d, r2, scale=ad2.scaling)
        cg.add(f"{prefix}w2.lora_b", (r2, d), cache["ax2"], dO, d, r2, ad2.scaling, d, 1)
    w1p, w2p = cache.get("w1p"), cache.get("w2p")
    if cache.get("repack"):  # the forward did not keep its packs (memory): re-pack this layer's active rows
        w1p, w2p = pack_active_rows2(lw.mlp.w1_t, lw.mlp.w2, nm)
    dz = torch.empty_like(a)
    _abi.call("lx_neuron_fc2_dgrad", dO.data_ptr(), B, s, d, f, blk, lw.mlp.w2.data_ptr(), nm.counts.data_ptr(),
              nm.ids.data_ptr(), _abi.ptr(dax2), _abi.ptr(ad2.a if ad2 else None), ad2.rank if ad2 else 0, a.data_ptr(),
              dz.data_ptr(), a.stride(0), _abi.ptr(w2p), _abi.ptr(cache.get("relu_bits")), st)
    if DEBUG_TAPS is not None:
        DEBUG_TAPS[f"{prefix}dO"], DEBUG_TAPS[f"{prefix}dz"] = dO, dz
    if ad2 is not None:
        cg.add(f"{prefix}w2.lora_a", (f, ad2.rank), dax2, a, f, ad2.rank, 1.0, 1, ad2.rank, masks=nm, blk=blk)
    if bitfit:
        cg.add(f"{prefix}b1", (f,), None, dz, f, 1, 1.0, 0, 1, masks=nm, blk=blk)
    dax1 = None
    if ad1 is not None:
        r1 = ad1.rank
        cg.add(f"{prefix}w1.lora_b", (r1, f), cache["ax1"], dz, f, r1, ad1.scaling, f, 1, masks=nm, blk=blk)
        if lp.get("b1") is not None:  # dz B1[:,cols]^T * s
            dax1 = rowproj_packed(dz, B, s, f, lp["b1"], r1, scale=ad1.scaling, masks=nm, blk=blk)
        else:
            dax1 = rowproj(dz, B, s, f, ad1.b, 1, f, r1, scale=ad1.scaling, masks=nm, blk=blk)
        cg.add(f"{prefix}w1.lora_a", (d, r1), dax1, x2, d, r1, 1.0, 1, r1)
    dx = torch.empty(B * s, d, dtype=torch.bfloat16, device=dev)
    _abi.call("lx_neuron_fc1_dgrad", dz.data_ptr(), dz.stride(0), B, s, d, f, blk, lw.mlp.w1_t.data_ptr(),
              nm.counts.data_ptr(), nm.ids.data_ptr(), _abi.ptr(dax1), _abi.ptr(ad1.a if ad1 else None),
              ad1.rank if ad1 else 0, dx.data_ptr(), 0, _abi.ptr(w1p), st)
    if own:
        cg.flush()
    return dx


def mha_backward(d_out, cache, lw: M.LayerWeights, lora: dict, dims: M.ModelDims, grads: dict, prefix: str = "",
                 bitfit: bool = False, cg: "_CgBatch | None" = None):
    """Backward of mha_forward (sf/autograd.py:127-162); score gradients only on active blocks.
    d_out [M, d] (bf16 preferred) -> dx bf16 [M, d]."""
    B, s = cache["n_items"], cache["s"]
    d, H, hd = dims.d_model, dims.n_heads, dims.head_dim
    dp = cache["dpool"]
    if cache["pidx"].shape[-1] != H:
        raise GradientError("cache layout head count does not match model dims")
    dev = cache["x"].device
    g = _bf16(d_out.reshape(-1, d)).contiguous()
    # output projection: d_heads = g Wo^T (+ LoRA(wo) fused), grads of wo's LoRA / bias
    ad_o = lora.get("wo")
    d_heads = M.proj_t(g, lw.wo)  # bf16
    dax_o = None
    if ad_o is not None:
        dax_o = rowproj(g, B, s, d, ad_o.b, 1, d, ad_o.rank, scale=ad_o.scaling)
        d_heads.addmm_(dax_o.to(torch.bfloat16), ad_o.a.t().to(torch.bfloat16))
    own = cg is None  # a caller-provided batch (block_backward) is flushed by the caller
    cg = _CgBatch(grads, B, s) if own else cg
    if ad_o is not None:
        r = ad_o.rank
        cg.add(f"{prefix}wo.lora_a", (d, r), dax_o, cache["o"], d, r, 1.0, 1, r)
        cg.add(f"{prefix}wo.lora_b", (r, d), cache["ax_o"], g, d, r, ad_o.scaling, d, 1)
    if bitfit:
        cg.add(f"{prefix}bo", (d,), None, g, d, 1, 1.0, 0, 1)
    qkv = cache["qkv"]
    ext = cache.get("ext", False)
    tq, r = cache["lora_t"], cache["lora_r"]
    kx = lw.lora_pack["kx"] if ext else 0
    # K-extended: dqkv_ext = [dq dk dv | dAx (bf16)], so one GEMM gives dqkv W^T + dAx A_cat^T
    dqkv_full = torch.empty(B * s, 3 * d + kx, dtype=torch.bfloat16, device=dev)
    dqkv = dqkv_full[:, : 3 * d] if ext else dqkv_full
    scale = 1.0 / float(np.sqrt(hd))
    attention_backward(qkv[:, :d], qkv[:, d : 2 * d], qkv[:, 2 * d :], cache["o"], d_heads, 3 * d, B, s, H, hd,
                       cache["pidx"], cache["stride"], dp, scale, cache["lse"], dqkv[:, :d], dqkv[:, d : 2 * d],
                       dqkv[:, 2 * d :])
    x2 = cache["x"]
    dax = None
    if tq:
        dax = torch.empty(B * s, len(tq) * r, dtype=torch.float32, device=dev)
        slots = [M.QKV_SLOT[t] for t in tq]
        bq = lw.lora_pack.get("b_qkv") if ext else None
        one = (bq is not None and d <= ROWPROJ_SEG_MAX_K and len({lora[t].scaling for t in tq}) == 1
               and all(b - a == slots[1] - slots[0] for a, b in zip(slots, slots[1:])))
        if one:
            # every target's dAx_t = dqkv[:, slot_t] B_t^T * s in one launch (equally spaced slots / packs / columns)
            rowproj_packed_seg(dqkv[:, slots[0] * d :], (slots[1] - slots[0]) * d if len(tq) > 1 else 0,
                                          d, bq, r, lora[tq[0]].scaling, dax, r, dqkv_full[:, 3 * d :], r, len(tq))
        for j, t in ([] if one else enumerate(tq)):
            ad, sl = lora[t], M.QKV_SLOT[t]
            if ext:
                rowproj_packed(dqkv[:, sl * d : (sl + 1) * d], B, s, d, lw.lora_pack["b"][t], r, scale=ad.scaling,
                               out=dax[:, j * r : (j + 1) * r], out_bf16=dqkv_full[:, 3 * d + j * r : 3 * d + (j + 1) * r])
            else:
                rowproj(dqkv[:, sl * d : (sl + 1) * d], B, s, d, ad.b, 1, d, r, scale=ad.scaling,
                        out=dax[:, j * r : (j + 1) * r])
    if ext:
        dx = M.proj_t(dqkv_full, lw.wqkv_ext[:d, :])
    else:
        # dx = dqkv W_qkv^T + dax A_cat^T (rank-n*r update)
        dx = M.proj_t(dqkv, lw.wqkv)
        if tq:
            dx.addmm_(dax.to(torch.bfloat16), cache["a_cat"].t().to(torch.bfloat16))
    for j, t in enumerate(tq):
        ad, sl = lora[t], M.QKV_SLOT[t]
        cg.add(f"{prefix}{t}.lora_a", (d, r), dax[:, j * r : (j + 1) * r], x2, d, r, 1.0, 1, r)
        cg.add(f"{prefix}{t}.lora_b", (r, d), cache["ax"][:, j * r : (j + 1) * r], dqkv[:, sl * d : (sl + 1) * d], d, r,
               ad.scaling, d, 1)
    if bitfit:
        for t in ("wq", "wk", "wv"):
            sl = M.QKV_SLOT[t]
            cg.add(f"{prefix}b{t[1]}", (d,), None, dqkv[:, sl * d : (sl + 1) * d], d, 1, 1.0, 0, 1)
    if own:
        cg.flush()
    return dx


def block_backward(d_out, model: M.Model, layer: int, cache, masks, grads: dict, d_out_bf16=None, inplace: bool = False,
                   cg: "_CgBatch | None" = None):
    """sf/autograd.py:165-181; d_out fp32 [B*s, d] (+ its bf16 copy). Returns (dx fp32, dx bf16).
    `cg`: a column-reduction batch shared with other layers (the caller flushes it); by default the
    layer's own batch is flushed here."""
    lw = model.weights.layers[layer]
    bitfit = model.peft_method == "bitfit"
    lora = {t: model.lora[(layer, t)] for t in model.lora_targets} if model.peft_method == "lora" else {}
    prefix = f"layers.{layer}."
    if DEBUG_TAPS is not None:
        DEBUG_TAPS[f"{prefix}d_out"] = d_out.clone()
    adapter = model.peft_method == "adapter"
    if d_out_bf16 is None:
        d_out_bf16 = d_out.to(torch.bfloat16)
    d_mlp = d_out_bf16
    if adapter:
        d_mlp = adapter_backward(d_out, model.adapters[(layer, "mlp")], cache["mlp_adapter"], grads, f"{prefix}mlp_adapter")
    nm = masks.neuron_mask if masks is not None else None
    # the layer's LoRA / BitFit column reductions (MLP then attention) run as one deterministic group
    # launch after both sublayers (their operands stay referenced by the batch until then)
    own = cg is None
    if own:
        cg = _CgBatch(grads, cache["mlp"]["n_items"], cache["mlp"]["s"])
    dh2 = mlp_backward(d_mlp, cache["mlp"], lw, lora, nm, model.dims, grads, prefix, bitfit, cg=cg)
    dy, dy_bf = layernorm_backward(dh2, cache["ln2"], accumulate_into=d_out if inplace else d_out.clone(), want_bf16=True)
    d_attn = dy_bf
    if adapter:
        d_attn = adapter_backward(dy, model.adapters[(layer, "attn")], cache["attn_adapter"], grads, f"{prefix}attn_adapter")
    dh1 = mha_backward(d_attn, cache["attn"], lw, lora, model.dims, grads, prefix, bitfit, cg=cg)
    if own:
        cg.flush()
    return layernorm_backward(dh1, cache["ln1"], accumulate_into=dy, want_bf16=True)


def model_backward(model: M.Model, cache, d_logits, masks=None) -> dict:
    """Full backward from dL/dlogits (sf/autograd.py:184-196); returns the GradientSet
    (summed over batch items)."""
    grads: dict = {}
    V = model.dims.vocab
    d_hf = M._mm_f32(d_logits.reshape(-1, V).to(torch.bfloat16), model.weights.emb)
    dh, dh_bf = layernorm_backward(d_hf, cache["lnf"], want_bf16=True)
    cg = None
    for k, layer in enumerate(reversed(range(model.dims.n_layers))):
        lm = None if masks is None else masks[layer]
        bc = cache["blocks"][layer]
        cg = cg or _CgBatch(grads, bc["mlp"]["n_items"], bc["mlp"]["s"])
        dh, dh_bf = block_backward(dh, model, layer, bc, lm, grads, dh_bf, inplace=True, cg=cg)
        if k % CG_LAYERS == CG_LAYERS - 1:  # CG_LAYERS layers' column reductions per group launch
            cg.flush()
            cg = None
    if cg is not None:
        cg.flush()
    for name, p in M.trainable_params(model).items():
        if name not in grads:
            grads[name] = torch.zeros_like(p)
    check_gradient_set(grads, model)
    return grads


def optimizer_step(state: M.PeftState, grads: dict, lr: float, betas=(0.9, 0.999), eps: float = 1e-8) -> M.PeftState:
    """In-place Adam over exactly the trainable set, float64 moments (sf/autograd.py:203-225)."""
    if set(grads) != set(state.params):
        missing = set(state.params) - set(grads)
        extra = set(grads) - set(state.params)
        raise GradientError(f"optimizer grads mismatch: missing={sorted(missing)}, extra={sorted(extra)}")
    b1, b2 = betas
    state.step += 1
    g = torch.empty_like(state.flat)
    for name, p in state.params.items():
        off = (p.data_ptr() - state.flat.data_ptr()) // 4
        g[off : off + p.numel()] = grads[name].reshape(-1)
    _abi.call("lx_adam_step", state.flat.data_ptr(), g.data_ptr(), state.m.data_ptr(), state.v.data_ptr(),
              state.flat.numel(), float(lr), float(b1), float(b2), float(eps), state.step,
              _abi.stream_handle(state.flat.device))
    return state


def adam_flat(p: torch.Tensor, g64: torch.Tensor, m: torch.Tensor, v: torch.Tensor, lr, b1, b2, eps, t) -> None:
    """Adam on the flat buffer with torch ops (float64 moments, sf/autograd.py:218-224): the test
    reference of lx_adam_step."""
    m.mul_(b1).add_(g64, alpha=1 - b1)
    v.mul_(b2).addcmul_(g64, g64, value=1 - b2)
    upd = (m / (1 - b1**t)) / ((v / (1 - b2**t)).sqrt_() + eps) * lr
    p.sub_(upd.to(p.dtype))
