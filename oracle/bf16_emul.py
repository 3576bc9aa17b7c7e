"""TEST INFRASTRUCTURE ONLY — the oracle model with the B200 path's rounding points.

`oracle/sf_oracle.py` restates the reference (sf/model.py, sf/autograd.py) in float32.
The device path computes the same algebra with bf16 operands and fp32 accumulation, and
rounds to bf16 at fixed points. On ill-conditioned fixtures (ReLU pre-activations within
bf16 resolution of 0, near-uniform attention whose q/k carry a large common mode) those
roundings move gradients by more than 1e-2 against float32, so a tight parity bar needs a
reference that rounds where the device rounds. This module is that reference: the same
per-sequence forward/backward as sf_oracle (each function cites the sf/ line it follows),
with `rd()` — round-to-nearest-even to bf16 — applied exactly at the device's rounding
points, and every GEMM evaluated in float64 on the rounded operands (the device's fp32
accumulation then differs only by accumulation order). With `exact=True` every `rd` is the
identity and the module reproduces sf_oracle (pinned by tests/test_bf16_emul.py).

Device rounding points (file:line of this repo's product path):
  * frozen weights W_q|W_k|W_v, W_o, W1, W2, emb and the q/k/v/o biases are bf16
    (model.py:from_arrays, model.py:_bias_bf16); b1, b2, LN parameters, LoRA A/B stay fp32;
  * the embedding gather reads bf16 emb (model.py:model_forward);
  * LN outputs h1, h2, hf are bf16 (csrc/layernorm.cu);
  * q/k/v = bf16(h1 W + bf16(h1 A) bf16(s B) + bf16(b)) in ONE rounding: the LoRA columns ride
    in the K-extended GEMM (model.py:mha_forward, ext path); W_o LoRA (not fused) rounds twice;
  * attention forward (csrc/attn_sm100.cu bsattn_fwd_tc_kernel): P = 2^(S c - m) with the lazy
    running max m over 128-key tiles, bf16(P) into P.V, fp32 row sum of the unrounded P,
    O = bf16(sum / l), lse = (m + log2 l) ln 2;
  * fc1 epilogue: a = bf16(relu(acc + b1 + s ax1 B1)) with ax1 = h2 A1 in fp32; fc2 epilogue:
    bf16(acc + b2 + s ax2 B2) (fp32 when an adapter follows), residual add in fp32 (next LN);
  * logits fp32 from bf16 hf and emb; d_logits is rounded to bf16 for the d_hf GEMM;
  * backward: LN backward fp32 with a bf16 copy feeding the GEMMs; dz = bf16((dO W2^T + dax2 A2^T)
    * (a > 0)); dx_mlp = bf16(dz W1^T + dax1 A1^T); d_heads = bf16(g W_o^T); attention backward
    recomputes P = 2^(S c - lse log2 e), dS = bf16(bf16(P) (dP - D)), D = rowsum(dO O),
    dV = bf16(bf16(P)^T dO), dK = bf16(c dS^T Q), dQ = bf16(c (dS K - eps kbar)) with eps the row
    sum of the bf16 dS and kbar the mean of the first 128 keys (the dQ kernel's common-mode correction); the q/k/v
    input-grad is one K-extended GEMM bf16(dq W_q^T + dk W_k^T + dv W_v^T + bf16(dax) bf16(A)^T);
  * LoRA / BitFit gradients are fp32 reductions of the bf16 activations and fp32 dax/ax;
  * Adapter: fp32 torch ops on the fp32 (or bf16-valued) inputs (model.py:adapter_forward).
"""

from __future__ import annotations

import numpy as np

from . import sf_oracle as O


def bf16(x) -> np.ndarray:
    """Round float32 values to the nearest bf16 (ties to even), returned as float32."""
    a = np.ascontiguousarray(np.asarray(x, dtype=np.float32))
    u = a.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32).reshape(a.shape)


class Emul:
    """Rounding policy: `rd` is bf16 rounding (device) or the identity (exact=True).

    `relu` (optional) teacher-forces the discrete ReLU decisions: {(layer, "mlp"): bool [s, F_act],
    (layer, "attn_ad") / (layer, "mlp_ad"): bool [s, r]} taken from the implementation under test. A
    pre-activation within accumulation-order noise of 0 can land on either side in two correct bf16
    implementations, and on ill-conditioned fixtures one such flip moves a gradient tensor by >1e-2; with
    the decisions shared, the comparison measures the continuous arithmetic only (like giving both sides
    the same neuron / attention masks)."""

    def __init__(self, exact: bool = False, relu: dict | None = None):
        self.exact = exact
        self.relu = relu or {}

    def rd(self, x):
        return np.asarray(x, np.float32) if self.exact else bf16(x)

    @staticmethod
    def mm(a, b):
        """GEMM on the given (already rounded) operands, float64 accumulate, fp32 result."""
        return (np.asarray(a, np.float64) @ np.asarray(b, np.float64)).astype(np.float32)


# ---------------------------------------------------------------------------------------- pieces


def _ln_fwd(e: Emul, x, g, b):
    y, c = O.layernorm_forward(x, g, b)  # sf/model.py:307-312, fp32 statistics
    return e.rd(y), c


def _fused_qkv(e: Emul, lw, lora):
    """q/k/v LoRA targets fused by K-extension (equal ranks, r % 8 == 0, n*r <= 16), model.py:ensure_lora_packs."""
    tq = [t for t in ("wq", "wk", "wv") if t in lora]
    ranks = {lora[t]["a"].shape[1] for t in tq}
    return bool(tq) and len(ranks) == 1 and next(iter(ranks)) % 8 == 0 and len(tq) * next(iter(ranks)) <= 16


def attention_forward_dev(e: Emul, q, k, v, coords, blk, scale, tile=128):
    """One head: sf/block_sparse.py sdd -> sparse_softmax -> dsd with the device kernel's numerics
    (lazy running max over key tiles, bf16 P into P.V, fp32 row sum). q, k, v already bf16-valued."""
    s, hd = q.shape
    mask = np.zeros((s, s), bool)
    for br, bc in np.asarray(coords).reshape(-1, 2):
        mask[br * blk : (br + 1) * blk, bc * blk : (bc + 1) * blk] = True
    S = e.mm(q, k.T)
    c = np.float32(scale * 1.4426950408889634)
    o = np.zeros((s, hd), np.float64)
    m = np.full(s, -np.inf, np.float32)
    l = np.zeros(s, np.float32)
    nt = -(-s // tile)
    for qt in range(nt):
        r0, r1 = qt * tile, min(s, (qt + 1) * tile)
        cols = [j for j in range(nt) if mask[r0:r1, j * tile : (j + 1) * tile].any()]
        for j in cols:
            c0, c1 = j * tile, min(s, (j + 1) * tile)
            Sb, Mb = S[r0:r1, c0:c1], mask[r0:r1, c0:c1]
            mx = np.where(Mb, Sb, -np.inf).max(1).astype(np.float32)
            with np.errstate(invalid="ignore", over="ignore"):  # rows with no active key yet: -inf - -inf
                mxs = (mx * c).astype(np.float32)
                mo = m[r0:r1]
                m_new = np.where(mxs > mo + 8.0, mxs, mo)  # lazy max (FA4-style, > 2^8 growth only)
                alpha = np.where(m_new == mo, 1.0, np.exp2(mo - m_new)).astype(np.float32)
                use = np.where(m_new == -np.inf, 0.0, m_new).astype(np.float32)
                p = np.where(Mb, np.exp2(Sb * c - use[:, None]), 0.0).astype(np.float32)
            l[r0:r1] = l[r0:r1] * alpha + p.sum(1, dtype=np.float32)
            o[r0:r1] = o[r0:r1] * alpha[:, None] + e.rd(p).astype(np.float64) @ v[c0:c1].astype(np.float64)
            m[r0:r1] = m_new
    inv = np.where(l > 0, 1.0 / np.maximum(l, 1e-30), 0.0)
    out = e.rd((o * inv[:, None]).astype(np.float32))
    lse = ((m + np.log2(np.maximum(l, 1e-30))) * np.float32(0.6931471805599453)).astype(np.float32)
    return out, lse, mask


def attention_backward_dev(e: Emul, q, k, v, o, do, lse, mask, scale):
    """One head: dsd_backward -> sparse_softmax_backward -> sdd_backward (sf/block_sparse.py:63-137)
    with the device kernels' numerics (bsattn_dkdv/dq kernels, csrc/attn_sm100.cu)."""
    c = np.float32(scale * 1.4426950408889634)
    S = e.mm(q, k.T)
    D = (o.astype(np.float64) * do.astype(np.float64)).sum(1).astype(np.float32)
    P = np.where(mask, np.exp2(S * c - (lse * np.float32(1.4426950408889634))[:, None]), 0.0).astype(np.float32)
    Pb = e.rd(P)
    dP = e.mm(do, v.T)
    dS = e.rd(np.where(mask, Pb * (dP - D[:, None]), 0.0))
    dv = e.rd(e.mm(Pb.T, do))
    dk = e.rd(e.mm(dS.T, q) * np.float32(scale))
    eps = dS.astype(np.float64).sum(1)
    kbar = k[: min(len(k), 128)].astype(np.float64).mean(0)  # the prep kernel's first-tile key mean
    dq_raw = dS.astype(np.float64) @ k.astype(np.float64)
    if not e.exact:
        dq_raw = dq_raw - eps[:, None] * kbar[None, :]  # the dQ kernel's row-sum (common-mode) correction
    dq = e.rd((dq_raw * scale).astype(np.float32))
    return dq, dk, dv


# ---------------------------------------------------------------------------------------- model


def mha_forward(e: Emul, x, lw, lora, head_patterns, pool, dims):
    """sf/model.py:322-360 at the device's rounding points; x = bf16 LN1 output."""
    d, hd, blk = dims.d_model, dims.head_dim, dims.attn_blk
    fused = _fused_qkv(e, lw, lora)
    cache = {"x": x, "fused": fused, "ax": {}}
    qkv = []
    for t, bn in (("wq", "bq"), ("wk", "bk"), ("wv", "bv")):
        z = e.mm(x, e.rd(lw[t])) + e.rd(lw[bn])
        ad = lora.get(t)
        if ad is not None:
            ax = e.mm(x, ad["a"])
            cache["ax"][t] = ax
            delta = e.mm(e.rd(ax), e.rd(ad["b"] * np.float32(ad["scaling"])))
            z = e.rd(z + delta) if fused else e.rd(e.rd(z) + delta)
        else:
            z = e.rd(z)
        qkv.append(z)
    q, k, v = qkv
    scale = 1.0 / np.sqrt(hd)
    heads = np.zeros_like(q)
    lses, masks = [], []
    for h, pid in enumerate(head_patterns):
        sl = slice(h * hd, (h + 1) * hd)
        oh, lse, mk = attention_forward_dev(e, q[:, sl], k[:, sl], v[:, sl], pool[pid], blk, scale)
        heads[:, sl] = oh
        lses.append(lse)
        masks.append(mk)
    out = e.rd(e.mm(heads, e.rd(lw["wo"])) + e.rd(lw["bo"]))
    ad = lora.get("wo")
    if ad is not None:
        ax = e.mm(heads, ad["a"])
        cache["ax"]["wo"] = ax
        out = e.rd(out + e.mm(e.rd(ax), e.rd(ad["b"] * np.float32(ad["scaling"]))))
    cache.update(q=q, k=k, v=v, heads=heads, lse=lses, masks=masks, patterns=list(head_patterns))
    return out, cache


def mha_backward(e: Emul, g, c, lw, lora, dims, grads, prefix, bitfit):
    """sf/autograd.py:127-162; g = bf16 dy."""
    d, hd = dims.d_model, dims.head_dim
    scale = 1.0 / np.sqrt(hd)
    ad_o = lora.get("wo")
    d_heads = e.rd(e.mm(g, e.rd(lw["wo"]).T))
    if ad_o is not None:
        dax_o = e.mm(g, ad_o["b"].T) * np.float32(ad_o["scaling"])
        d_heads = e.rd(d_heads + e.mm(e.rd(dax_o), e.rd(ad_o["a"].T)))
        O._acc(grads, f"{prefix}wo.lora_a", e.mm(c["heads"].T, dax_o))
        O._acc(grads, f"{prefix}wo.lora_b", np.float32(ad_o["scaling"]) * e.mm(c["ax"]["wo"].T, g))
    if bitfit:
        O._acc(grads, f"{prefix}bo", g.astype(np.float64).sum(0).astype(np.float32))
    q, k, v = c["q"], c["k"], c["v"]
    dq, dk, dv = np.zeros_like(q), np.zeros_like(k), np.zeros_like(v)
    for h in range(len(c["patterns"])):
        sl = slice(h * hd, (h + 1) * hd)
        dq[:, sl], dk[:, sl], dv[:, sl] = attention_backward_dev(e, q[:, sl], k[:, sl], v[:, sl], c["heads"][:, sl],
                                                                 d_heads[:, sl], c["lse"][h], c["masks"][h], scale)
    dx = e.mm(dq, e.rd(lw["wq"]).T) + e.mm(dk, e.rd(lw["wk"]).T) + e.mm(dv, e.rd(lw["wv"]).T)
    for t, dt, bn in (("wq", dq, "bq"), ("wk", dk, "bk"), ("wv", dv, "bv")):
        ad = lora.get(t)
        if ad is not None:
            dax = e.mm(dt, ad["b"].T) * np.float32(ad["scaling"])
            O._acc(grads, f"{prefix}{t}.lora_a", e.mm(c["x"].T, dax))
            O._acc(grads, f"{prefix}{t}.lora_b", np.float32(ad["scaling"]) * e.mm(c["ax"][t].T, dt))
            dx = dx + e.mm(e.rd(dax), e.rd(ad["a"]).T)
        if bitfit:
            O._acc(grads, f"{prefix}{bn}", dt.astype(np.float64).sum(0).astype(np.float32))
    return e.rd(dx)


def mlp_forward(e: Emul, x, lw, lora, neuron_mask, dims, out_f32=False, layer=None):
    """sf/model.py:363-400 at the device's rounding points; x = bf16 LN2 output."""
    _, cols = O.active_columns(neuron_mask, dims.d_ff, dims.blk_size)
    z = e.mm(x, e.rd(lw["w1"])[:, cols]) + lw["b1"][cols]
    ad1, ad2 = lora.get("w1"), lora.get("w2")
    ax1 = ax2 = None
    if ad1 is not None and cols.size:
        ax1 = e.mm(x, ad1["a"])
        z = z + np.float32(ad1["scaling"]) * e.mm(ax1, ad1["b"][:, cols])
    act = z > 0
    forced = e.relu.get((layer, "mlp"))
    if forced is not None:
        act = np.asarray(forced, bool)[:, : z.shape[1]]
    a = e.rd(np.where(act, z, 0))
    out = e.mm(a, e.rd(lw["w2"])[cols, :]) + lw["b2"]
    if ad2 is not None and cols.size:
        ax2 = e.mm(a, ad2["a"][cols, :])
        out = out + np.float32(ad2["scaling"]) * e.mm(ax2, ad2["b"])
    out = out.astype(np.float32) if out_f32 else e.rd(out)
    return out, {"x": x, "z": z, "a": a, "act": act, "cols": cols, "ax1": ax1, "ax2": ax2}


def mlp_backward(e: Emul, dO, c, lw, lora, dims, grads, prefix, bitfit):
    """sf/autograd.py:78-124; dO bf16-valued."""
    cols, x, a = c["cols"], c["x"], c["a"]
    if bitfit:
        O._acc(grads, f"{prefix}b2", dO.astype(np.float64).sum(0).astype(np.float32))
    da = e.mm(dO, e.rd(lw["w2"])[cols, :].T) if cols.size else np.zeros_like(a)
    ad2, ad1 = lora.get("w2"), lora.get("w1")
    if ad2 is not None and cols.size:
        dax2 = e.mm(dO, ad2["b"].T) * np.float32(ad2["scaling"])
        O._acc(grads, f"{prefix}w2.lora_b", np.float32(ad2["scaling"]) * e.mm(c["ax2"].T, dO))
        gA = np.zeros_like(ad2["a"])
        gA[cols, :] = e.mm(a.T, dax2)
        O._acc(grads, f"{prefix}w2.lora_a", gA)
        da = da + e.mm(dax2, ad2["a"][cols, :].T)
    elif ad2 is not None:
        O._acc(grads, f"{prefix}w2.lora_b", np.zeros_like(ad2["b"]))
        O._acc(grads, f"{prefix}w2.lora_a", np.zeros_like(ad2["a"]))
    dz = e.rd(da * c["act"])
    c["dO"], c["dz"] = dO, dz  # diagnostics (tools/debug_bitfit.py)
    if bitfit:
        gb = np.zeros_like(lw["b1"])
        if cols.size:
            gb[cols] = dz.astype(np.float64).sum(0)
        O._acc(grads, f"{prefix}b1", gb)
    dx = e.mm(dz, e.rd(lw["w1"])[:, cols].T) if cols.size else np.zeros_like(x)
    if ad1 is not None:
        gb = np.zeros_like(ad1["b"])
        if cols.size:
            gb[:, cols] = np.float32(ad1["scaling"]) * e.mm(c["ax1"].T, dz)
            dax1 = e.mm(dz, ad1["b"][:, cols].T) * np.float32(ad1["scaling"])
            O._acc(grads, f"{prefix}w1.lora_a", e.mm(x.T, dax1))
            dx = dx + e.mm(dax1, ad1["a"].T)
        else:
            O._acc(grads, f"{prefix}w1.lora_a", np.zeros_like(ad1["a"]))
        O._acc(grads, f"{prefix}w1.lora_b", gb)
    return e.rd(dx)


def adapter_forward(e: Emul, x, ad, key=None):
    """sf/model.py:315-319 (fp32 on the device too), ReLU decisions optionally teacher-forced."""
    x = x.astype(np.float32)
    z = e.mm(x, ad["w_down"]) + ad["b_down"]
    act = z > 0
    forced = e.relu.get(key)
    if forced is not None:
        act = np.asarray(forced, bool)
    h = np.where(act, z, 0).astype(np.float32)
    return x + e.mm(h, ad["w_up"]) + ad["b_up"], {"x": x, "z": z, "h": h, "act": act}


def adapter_backward(e: Emul, dy, ad, c, grads, prefix):
    """sf/autograd.py:69-75 (fp32)."""
    O._acc(grads, f"{prefix}.w_up", e.mm(c["h"].T, dy))
    O._acc(grads, f"{prefix}.b_up", dy.astype(np.float64).sum(0).astype(np.float32))
    dh = e.mm(dy, ad["w_up"].T) * c["act"]
    O._acc(grads, f"{prefix}.w_down", e.mm(c["x"].T, dh))
    O._acc(grads, f"{prefix}.b_down", dh.astype(np.float64).sum(0).astype(np.float32))
    return dy + e.mm(dh, ad["w_down"].T)


def block_forward(e: Emul, m: O.OModel, i: int, h, masks_i):
    """sf/model.py:403-433: one pre-LN block on the fp32 residual h [s, d]; masks_i = (head_patterns, neuron_mask)."""
    lw, lora = m.layers[i], O._layer_lora(m, i)
    adapter = m.peft == "adapter"
    pats, nm = masks_i
    h1, c1 = _ln_fwd(e, h, lw["ln1_g"], lw["ln1_b"])
    att, ca = mha_forward(e, h1, lw, lora, pats, m.pool, m.dims)
    caa = None
    if adapter:
        att, caa = adapter_forward(e, att, m.adapters[(i, "attn")], (i, "attn_ad"))
    y = h + att
    h2, c2 = _ln_fwd(e, y, lw["ln2_g"], lw["ln2_b"])
    mo, cm = mlp_forward(e, h2, lw, lora, nm, m.dims, out_f32=adapter, layer=i)
    cma = None
    if adapter:
        mo, cma = adapter_forward(e, mo, m.adapters[(i, "mlp")], (i, "mlp_ad"))
    return y + mo, {"ln1": c1, "attn": ca, "attn_ad": caa, "ln2": c2, "mlp": cm, "mlp_ad": cma}


def block_backward(e: Emul, m: O.OModel, i: int, c, dh, grads: dict):
    """sf/autograd.py:165-181: fp32 d_out of block i -> fp32 d_in; accumulates the block's trainable gradients."""
    lw, lora, prefix = m.layers[i], O._layer_lora(m, i), f"layers.{i}."
    adapter, bitfit = m.peft == "adapter", m.peft == "bitfit"
    dm = dh
    if adapter:
        dm = adapter_backward(e, dh, m.adapters[(i, "mlp")], c["mlp_ad"], grads, f"{prefix}mlp_adapter")
    dh2 = mlp_backward(e, e.rd(dm), c["mlp"], lw, lora, m.dims, grads, prefix, bitfit)
    dy = dh + O.layernorm_backward(dh2, c["ln2"])
    da = dy
    if adapter:
        da = adapter_backward(e, dy, m.adapters[(i, "attn")], c["attn_ad"], grads, f"{prefix}attn_adapter")
    dh1 = mha_backward(e, e.rd(da), c["attn"], lw, lora, m.dims, grads, prefix, bitfit)
    return dy + O.layernorm_backward(dh1, c["ln1"])


def model_forward(e: Emul, m: O.OModel, tokens, masks):
    """sf/model.py:436-451 for one sequence; masks = list of (head_patterns, neuron_mask)."""
    emb = e.rd(m.emb)
    h = emb[tokens].astype(np.float32)
    caches = []
    for i in range(m.dims.n_layers):
        h, c = block_forward(e, m, i, h, masks[i])
        caches.append(c)
    hf, cf = _ln_fwd(e, h, m.lnf_g, m.lnf_b)
    return e.mm(hf, emb.T), {"blocks": caches, "lnf": cf}


def model_backward(e: Emul, m: O.OModel, cache, d_logits):
    """sf/autograd.py:184-196."""
    grads = {}
    emb = e.rd(m.emb)
    dh = O.layernorm_backward(e.mm(e.rd(d_logits), emb), cache["lnf"])
    for i in reversed(range(m.dims.n_layers)):
        dh = block_backward(e, m, i, cache["blocks"][i], dh, grads)
    for name, p in O.trainable_params(m).items():
        if name not in grads:
            grads[name] = np.zeros_like(p)
    return grads
