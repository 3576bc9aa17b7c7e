"""Hand-written backward for the trainable set only (drop-in for sf/autograd.py).

Inactive neuron blocks and attention blocks are never touched: the MLP
input-grad runs the tcgen05 gather-GEMMs over the forward's index lists, the
LoRA / BitFit gradients are deterministic skinny reductions over the packed
active columns (inactive rows/columns stay exactly 0, sf/autograd.py:89-90),
and attention gradients flow through the block-sparse backward kernels only.
Gradients are sums over the batch items (the reference harness sums per-item
gradients and divides by the batch size, sf/harness.py:413-415).
"""

from __future__ import annotations

import numpy as np
import torch

from . import model as M
from .block_sparse import attention_backward
from .errors import GradientError
from .neuron_ops import colgrad, rowproj
from . import _abi


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


def lora_linear_backward(dz, w, adapter, cache, grads: dict, prefix: str, bias_name):
    """sf/autograd.py:48-58; dz fp32 [M, d_out], w bf16 [d_in, d_out]. Returns dx fp32."""
    dx = M._mm_f32(dz.to(torch.bfloat16), w.t())
    if adapter is not None:
        d_ax = (dz @ adapter.b.t()) * adapter.scaling
        _acc(grads, f"{prefix}.lora_a", cache["x"].float().t() @ d_ax)
        _acc(grads, f"{prefix}.lora_b", adapter.scaling * (cache["ax"].t() @ dz))
        dx.addmm_(d_ax, adapter.a.t())
    if bias_name is not None:
        _acc(grads, bias_name, dz.sum(0))
    return dx


def layernorm_backward(dy, cache, accumulate_into: torch.Tensor | None = None) -> torch.Tensor:
    """sf/autograd.py:61-66 on the fused kernel: returns (accumulate_into or 0) + LN'(dy) (fp32)."""
    x = cache["x"]
    Mr, d = x.shape
    out = accumulate_into if accumulate_into is not None else torch.zeros(Mr, d, dtype=torch.float32, device=x.device)
    dy2 = dy.reshape(Mr, d).contiguous()
    _abi.call("lx_layernorm_bwd", dy2.data_ptr(), int(dy2.dtype == torch.float32), x.data_ptr(), cache["gamma"].data_ptr(),
              cache["mean"].data_ptr(), cache["inv_std"].data_ptr(), Mr, d, out.data_ptr(), _abi.stream_handle(x.device))
    return out


def adapter_backward(dy, ad: M.AdapterLayer, cache, grads: dict, prefix: str):
    """sf/autograd.py:69-75 (fp32)."""
    _acc(grads, f"{prefix}.w_up", cache["h"].t() @ dy)
    _acc(grads, f"{prefix}.b_up", dy.sum(0))
    dh = (dy @ ad.w_up.t()) * (cache["z"] > 0)
    _acc(grads, f"{prefix}.w_down", cache["x"].t() @ dh)
    _acc(grads, f"{prefix}.b_down", dh.sum(0))
    return dy + dh @ ad.w_down.t()


def mlp_backward(d_out, cache, lw: M.LayerWeights, lora: dict, neuron_mask, dims: M.ModelDims, grads: dict,
                 prefix: str = "", bitfit: bool = False):
    """Backward of mlp_forward (sf/autograd.py:78-124). d_out fp32/bf16 [M, d] -> dx fp32 [M, d]."""
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
    dO = d_out.reshape(-1, d).to(torch.bfloat16).contiguous()
    st = _abi.stream_handle(dev)
    if bitfit:
        _acc(grads, f"{prefix}b2", colgrad(None, dO, B, s, d, 1, 1.0, torch.empty(d, device=dev), 0, 1))
    ad1, ad2 = lora.get("w1"), lora.get("w2")
    dax2 = None
    if ad2 is not None:
        r2 = ad2.rank
        dax2 = rowproj(dO, B, s, d, ad2.b, 1, d, r2, scale=ad2.scaling)  # dO B2^T * s
        _acc(grads, f"{prefix}w2.lora_b", colgrad(cache["ax2"], dO, B, s, d, r2, ad2.scaling,
                                                   torch.empty(r2, d, device=dev), d, 1))
    dz = torch.empty_like(a)
    _abi.call("lx_neuron_fc2_dgrad", dO.data_ptr(), B, s, d, f, blk, lw.mlp.w2.data_ptr(), nm.counts.data_ptr(),
              nm.ids.data_ptr(), _abi.ptr(dax2), _abi.ptr(ad2.a if ad2 else None), ad2.rank if ad2 else 0, a.data_ptr(),
              dz.data_ptr(), a.stride(0), st)
    if ad2 is not None:
        _acc(grads, f"{prefix}w2.lora_a", colgrad(dax2, a, B, s, f, ad2.rank, 1.0, torch.empty(f, ad2.rank, device=dev),
                                                  1, ad2.rank, masks=nm, blk=blk))
    if bitfit:
        _acc(grads, f"{prefix}b1", colgrad(None, dz, B, s, f, 1, 1.0, torch.empty(f, device=dev), 0, 1, masks=nm, blk=blk))
    dax1 = None
    if ad1 is not None:
        r1 = ad1.rank
        _acc(grads, f"{prefix}w1.lora_b", colgrad(cache["ax1"], dz, B, s, f, r1, ad1.scaling,
                                                   torch.empty(r1, f, device=dev), f, 1, masks=nm, blk=blk))
        dax1 = rowproj(dz, B, s, f, ad1.b, 1, f, r1, scale=ad1.scaling, masks=nm, blk=blk)  # dz B1[:,cols]^T * s
        _acc(grads, f"{prefix}w1.lora_a", colgrad(dax1, x2, B, s, d, r1, 1.0, torch.empty(d, r1, device=dev), 1, r1))
    dx = torch.empty(B * s, d, dtype=torch.bfloat16, device=dev)
    _abi.call("lx_neuron_fc1_dgrad", dz.data_ptr(), dz.stride(0), B, s, d, f, blk, lw.mlp.w1_t.data_ptr(),
              nm.counts.data_ptr(), nm.ids.data_ptr(), _abi.ptr(dax1), _abi.ptr(ad1.a if ad1 else None),
              ad1.rank if ad1 else 0, dx.data_ptr(), st)
    return dx


def mha_backward(d_out, cache, lw: M.LayerWeights, lora: dict, dims: M.ModelDims, grads: dict, prefix: str = "",
                 bitfit: bool = False):
    """Backward of mha_forward (sf/autograd.py:127-162); score gradients only on active blocks."""
    B, s = cache["n_items"], cache["s"]
    d, H, hd = dims.d_model, dims.n_heads, dims.head_dim
    dp = cache["dpool"]
    if cache["pidx"].shape[-1] != H:
        raise GradientError("cache layout head count does not match model dims")
    d_heads = lora_linear_backward(d_out.reshape(-1, d).float(), lw.wo, lora.get("wo"), cache["co"], grads,
                                   f"{prefix}wo", f"{prefix}bo" if bitfit else None)
    qkv = cache["qkv"]
    d_o = d_heads.to(torch.bfloat16)
    dqkv = torch.empty_like(qkv)
    scale = 1.0 / float(np.sqrt(hd))
    attention_backward(qkv[:, :d], qkv[:, d : 2 * d], qkv[:, 2 * d :], cache["o"], d_o, 3 * d, B, s, H, hd,
                       cache["pidx"], cache["stride"], dp, scale, cache["lse"], dqkv[:, :d], dqkv[:, d : 2 * d],
                       dqkv[:, 2 * d :])
    x2 = cache["x"]
    dx = M._mm_f32(dqkv, lw.wqkv.t())
    for j, t in enumerate(("wq", "wk", "wv")):
        sl = dqkv[:, j * d : (j + 1) * d]
        ad = lora.get(t)
        if ad is not None:
            g = sl.float()
            d_ax = (g @ ad.b.t()) * ad.scaling
            _acc(grads, f"{prefix}{t}.lora_a", x2.float().t() @ d_ax)
            _acc(grads, f"{prefix}{t}.lora_b", ad.scaling * (cache["ax"][t].t() @ g))
            dx.addmm_(d_ax, ad.a.t())
        if bitfit:
            _acc(grads, f"{prefix}b{t[1]}", sl.float().sum(0))
    return dx


def block_backward(d_out, model: M.Model, layer: int, cache, masks, grads: dict):
    """sf/autograd.py:165-181; d_out fp32 [B*s, d]."""
    lw = model.weights.layers[layer]
    bitfit = model.peft_method == "bitfit"
    lora = {t: model.lora[(layer, t)] for t in model.lora_targets} if model.peft_method == "lora" else {}
    prefix = f"layers.{layer}."
    d_mlp = d_out
    if model.peft_method == "adapter":
        d_mlp = adapter_backward(d_out, model.adapters[(layer, "mlp")], cache["mlp_adapter"], grads, f"{prefix}mlp_adapter")
    nm = masks.neuron_mask if masks is not None else None
    dh2 = mlp_backward(d_mlp, cache["mlp"], lw, lora, nm, model.dims, grads, prefix, bitfit)
    dy = layernorm_backward(dh2, cache["ln2"], accumulate_into=d_out.clone())
    d_attn = dy
    if model.peft_method == "adapter":
        d_attn = adapter_backward(dy, model.adapters[(layer, "attn")], cache["attn_adapter"], grads, f"{prefix}attn_adapter")
    dh1 = mha_backward(d_attn, cache["attn"], lw, lora, model.dims, grads, prefix, bitfit)
    return layernorm_backward(dh1, cache["ln1"], accumulate_into=dy)


def model_backward(model: M.Model, cache, d_logits, masks=None) -> dict:
    """Full backward from dL/dlogits (sf/autograd.py:184-196); returns the GradientSet
    (summed over batch items)."""
    grads: dict = {}
    V = model.dims.vocab
    d_hf = M._mm_f32(d_logits.reshape(-1, V).to(torch.bfloat16), model.weights.emb)
    dh = layernorm_backward(d_hf, cache["lnf"])
    for layer in reversed(range(model.dims.n_layers)):
        lm = None if masks is None else masks[layer]
        dh = block_backward(dh, model, layer, cache["blocks"][layer], lm, grads)
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
    t = state.step
    if state.flat is not None:
        g = torch.empty_like(state.m)
        for name, p in state.params.items():
            off = p.data_ptr() - state.flat.data_ptr()
            g[off // 4 : off // 4 + p.numel()] = grads[name].reshape(-1).double()
        adam_flat(state.flat, g, state.m, state.v, lr, b1, b2, eps, t)
        return state
    for name, p in state.params.items():  # pragma: no cover - flat path is the default
        g = grads[name].double()
        m = state.m.setdefault(name, torch.zeros_like(g))
        v = state.v.setdefault(name, torch.zeros_like(g))
        m.mul_(b1).add_(g, alpha=1 - b1)
        v.mul_(b2).addcmul_(g, g, value=1 - b2)
        p -= (lr * (m / (1 - b1**t)) / ((v / (1 - b2**t)).sqrt() + eps)).to(p.dtype)
    return state


def adam_flat(p: torch.Tensor, g64: torch.Tensor, m: torch.Tensor, v: torch.Tensor, lr, b1, b2, eps, t) -> None:
    """Adam on the flat buffer (float64 moments), same update order as sf/autograd.py:218-224."""
    m.mul_(b1).add_(g64, alpha=1 - b1)
    v.mul_(b2).addcmul_(g64, g64, value=1 - b2)
    upd = (m / (1 - b1**t)) / ((v / (1 - b2**t)).sqrt_() + eps) * lr
    p.sub_(upd.to(p.dtype))
