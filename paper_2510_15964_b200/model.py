"""Frozen-backbone transformer with LoRA / Adapter / BitFit on the B200
(drop-in for sf/model.py).

Semantics mirror the reference exactly: pre-LN residual blocks, non-causal
block-sparse attention without positional embedding (sf/model.py:443), ReLU
MLP restricted to active neuron blocks, tied unembedding, mean cross-entropy.
Every forward takes a batch of items [B, s] at once (the reference loops over
sequences, sf/harness.py:401-411); masks stay per item, so results equal the
per-item loop and gradients equal the reference's per-item sum.

Device layout: residual stream fp32 [B*s, d]; LN outputs and GEMM operands
bf16; frozen weights bf16 (W_qkv fused [d, 3d]; W1^T and W2 [d_ff, d]);
trainable tensors fp32 views into one flat buffer (`PeftState`) so the
data-parallel all-reduce is a single NCCL call.

Hot-path kernels: mask build (predictor.py), neuron-sparse MLP (neuron_ops.py),
block-sparse attention (block_sparse.py), LayerNorm (+ fused predictor
downsample). Dense neighbours (Q/K/V/O projections, LM head) use cuBLAS.
"""

from __future__ import annotations

import copy
import hashlib
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _abi, neuron_ops
from .block_sparse import attention_forward
from .errors import ShapeError
from .neuron_ops import LayeredWeights, NeuronMasks, lower_mask, rowproj, rowproj_packed
from .patterns import DevicePool, LayoutTable, build_pool, device_pool

LORA_TARGET_SHAPES = {"wq": "attn", "wk": "attn", "wv": "attn", "wo": "attn", "w1": "mlp_in", "w2": "mlp_out"}
PEFT_METHODS = ("lora", "adapter", "bitfit")
BIAS_NAMES = ("bq", "bk", "bv", "bo", "b1", "b2")


@dataclass(frozen=True)
class ModelDims:
    """sf/model.py:33-60."""

    d_model: int
    n_heads: int
    d_ff: int
    seq_len: int
    n_layers: int = 4
    vocab: int = 256
    blk_size: int = 16
    attn_blk: int = 16

    def __post_init__(self):
        if self.d_model % self.n_heads:
            raise ShapeError(f"d_model {self.d_model} not divisible by n_heads {self.n_heads}")
        if self.seq_len % self.attn_blk:
            raise ShapeError(f"seq_len {self.seq_len} not divisible by attn_blk {self.attn_blk}")

    @property
    def head_dim(self) -> int:
        return self.d_model // self.n_heads

    @property
    def n_blk(self) -> int:
        return neuron_ops.n_blocks(self.d_ff, self.blk_size)

    @property
    def n_b(self) -> int:
        return self.seq_len // self.attn_blk


@dataclass
class LoraAdapter:
    """z = xW + scaling * (xA)B; a (d_in, r), b (r, d_out) fp32 (sf/model.py:63-73)."""

    a: torch.Tensor
    b: torch.Tensor
    scaling: float = 1.0

    @property
    def rank(self) -> int:
        return self.a.shape[1]


@dataclass
class AdapterLayer:
    """Bottleneck adapter x + relu(x Wd + bd) Wu + bu (sf/model.py:76-83)."""

    w_down: torch.Tensor
    b_down: torch.Tensor
    w_up: torch.Tensor
    b_up: torch.Tensor


@dataclass
class LayerWeights:
    """sf/model.py:86-102 with the device layout described in the module docstring."""

    wqkv: torch.Tensor  # bf16 [d, 3d]
    wo: torch.Tensor  # bf16 [d, d]
    bqkv: torch.Tensor  # fp32 [3d] (bq | bk | bv)
    bo: torch.Tensor
    mlp: LayeredWeights
    b1: torch.Tensor
    b2: torch.Tensor
    ln1_g: torch.Tensor
    ln1_b: torch.Tensor
    ln2_g: torch.Tensor
    ln2_b: torch.Tensor
    # K-extended q/k/v projection [d + kx, 3d + kx] (wqkv is its [:d, :3d] view): rows d.. hold s*B of the
    # LoRA targets, columns 3d.. hold their A, so one GEMM applies x W + s (xA) B and one dx GEMM adds
    # dAx A^T (sf/model.py:292-304, sf/autograd.py:48-58). Set by ensure_lora_packs.
    wqkv_ext: torch.Tensor | None = None
    lora_pack: dict | None = None

    @property
    def d(self) -> int:
        return self.wo.shape[0]

    @property
    def bq(self):
        return self.bqkv[: self.d]

    @property
    def bk(self):
        return self.bqkv[self.d : 2 * self.d]

    @property
    def bv(self):
        return self.bqkv[2 * self.d :]

    @property
    def wq(self):
        return self.wqkv[:, : self.d]

    @property
    def wk(self):
        return self.wqkv[:, self.d : 2 * self.d]

    @property
    def wv(self):
        return self.wqkv[:, 2 * self.d :]


@dataclass
class FrozenWeights:
    emb: torch.Tensor  # bf16 [V, d] (tied embedding / unembedding)
    layers: list
    lnf_g: torch.Tensor
    lnf_b: torch.Tensor


@dataclass
class PeftState:
    """Trainable set with Adam moments (sf/model.py:113-127). `params` are views of
    one flat fp32 buffer; moments are float64 like the reference."""

    method: str
    params: dict
    flat: torch.Tensor | None = None
    m: torch.Tensor | None = None
    v: torch.Tensor | None = None
    step: int = 0


@dataclass
class LayerMasks:
    """sf/model.py:130-133. head_patterns: list[str] (shared) or int32 [B, H] pool indices;
    neuron_mask: bool [n_blk] / [B, n_blk] or NeuronMasks."""

    head_patterns: object
    neuron_mask: object


def dense_masks(dims: ModelDims) -> list[LayerMasks]:
    return [LayerMasks(["dense"] * dims.n_heads, np.ones(dims.n_blk, dtype=bool)) for _ in range(dims.n_layers)]


@dataclass
class Model:
    dims: ModelDims
    weights: FrozenWeights
    pool: dict
    peft_method: str
    lora: dict = field(default_factory=dict)
    adapters: dict = field(default_factory=dict)
    lora_targets: tuple = ()
    device: torch.device = torch.device("cuda")
    _dpool: DevicePool | None = None

    @property
    def dpool(self) -> DevicePool:
        if self._dpool is None:
            self._dpool = device_pool(self.pool, self.device, self.dims.seq_len, self.dims.attn_blk)
        return self._dpool


# ---------------------------------------------------------------- construction


def _t(a, device, dtype=torch.float32):
    return torch.as_tensor(np.asarray(a) if not torch.is_tensor(a) else a).to(device=device, dtype=dtype).contiguous()


def from_arrays(dims: ModelDims, peft: str, emb, layers: list[dict], lnf_g, lnf_b, lora: dict | None = None,
                adapters: dict | None = None, lora_targets=(), device="cuda") -> Model:
    """Build a device model from reference-format arrays (w1 is [d, d_ff]; lora values have
    a/b/scaling; adapters have w_down/b_down/w_up/b_up)."""
    dev = torch.device(device)
    L = []
    for lw in layers:
        L.append(LayerWeights(
            wqkv=torch.cat([_t(lw["wq"], dev), _t(lw["wk"], dev), _t(lw["wv"], dev)], 1).to(torch.bfloat16).contiguous(),
            wo=_t(lw["wo"], dev, torch.bfloat16),
            bqkv=torch.cat([_t(lw["bq"], dev), _t(lw["bk"], dev), _t(lw["bv"], dev)]).contiguous(),
            bo=_t(lw["bo"], dev), mlp=LayeredWeights.from_row_major(np.asarray(lw["w1"]) if not torch.is_tensor(lw["w1"]) else lw["w1"],
                                                                   np.asarray(lw["w2"]) if not torch.is_tensor(lw["w2"]) else lw["w2"], dev),
            b1=_t(lw["b1"], dev), b2=_t(lw["b2"], dev), ln1_g=_t(lw["ln1_g"], dev), ln1_b=_t(lw["ln1_b"], dev),
            ln2_g=_t(lw["ln2_g"], dev), ln2_b=_t(lw["ln2_b"], dev)))
    m = Model(dims, FrozenWeights(_t(emb, dev, torch.bfloat16), L, _t(lnf_g, dev), _t(lnf_b, dev)), build_pool(dims.n_b), peft,
              lora_targets=tuple(lora_targets) if peft == "lora" else (), device=dev)
    for key, ad in (lora or {}).items():
        m.lora[key] = LoraAdapter(_t(ad["a"], dev), _t(ad["b"], dev), float(ad.get("scaling", 1.0)))
    for key, ad in (adapters or {}).items():
        m.adapters[key] = AdapterLayer(*(_t(ad[k], dev) for k in ("w_down", "b_down", "w_up", "b_up")))
    return m


def build_model(dims: ModelDims, seed: int, peft: str = "lora", lora_rank: int = 8,
                lora_targets: tuple = ("wq", "wv", "w1", "w2"), adapter_rank: int = 8, init_scale: float = 0.02,
                device="cuda") -> Model:
    """Random-init model with the reference's init distribution (sf/model.py:174-231):
    projections / embedding / LoRA-A / adapter-down N(0, init_scale^2), zero biases,
    LN gamma=1 beta=0, LoRA-B and adapter-up zero. Drawn on the device (torch
    generator); use `from_arrays` to load reference-initialised weights."""
    if peft not in PEFT_METHODS:
        raise ValueError(f"unknown peft method {peft!r}")
    dev = torch.device(device)
    g = torch.Generator(device=dev).manual_seed(seed)
    d, f = dims.d_model, dims.d_ff

    def rn(*shape, dtype=torch.bfloat16):
        return (torch.randn(*shape, generator=g, device=dev) * init_scale).to(dtype)

    z = lambda n: torch.zeros(n, device=dev)  # noqa: E731
    layers = [LayerWeights(rn(d, 3 * d), rn(d, d), z(3 * d), z(d), LayeredWeights(rn(f, d), rn(f, d)), z(f), z(d),
                           torch.ones(d, device=dev), z(d), torch.ones(d, device=dev), z(d)) for _ in range(dims.n_layers)]
    m = Model(dims, FrozenWeights(rn(dims.vocab, d), layers, torch.ones(d, device=dev), z(d)), build_pool(dims.n_b), peft,
              lora_targets=tuple(lora_targets) if peft == "lora" else (), device=dev)
    shapes = {"attn": (d, d), "mlp_in": (d, f), "mlp_out": (f, d)}
    if peft == "lora":
        for i in range(dims.n_layers):
            for t in m.lora_targets:
                di, do = shapes[LORA_TARGET_SHAPES[t]]
                m.lora[(i, t)] = LoraAdapter(rn(di, lora_rank, dtype=torch.float32), torch.zeros(lora_rank, do, device=dev))
    elif peft == "adapter":
        for i in range(dims.n_layers):
            for sub in ("attn", "mlp"):
                m.adapters[(i, sub)] = AdapterLayer(rn(d, adapter_rank, dtype=torch.float32), z(adapter_rank),
                                                    torch.zeros(adapter_rank, d, device=dev), z(d))
    return m


def _param_slots(model: Model) -> list[tuple[str, object, str]]:
    """(name, owner, attribute) in the reference's trainable order (sf/model.py:234-249)."""
    out = []
    if model.peft_method == "lora":
        for (i, t), ad in sorted(model.lora.items()):
            out += [(f"layers.{i}.{t}.lora_a", ad, "a"), (f"layers.{i}.{t}.lora_b", ad, "b")]
    elif model.peft_method == "adapter":
        for (i, sub), ad in sorted(model.adapters.items()):
            out += [(f"layers.{i}.{sub}_adapter.{k}", ad, k) for k in ("w_down", "b_down", "w_up", "b_up")]
    else:
        for i, lw in enumerate(model.weights.layers):
            out += [(f"layers.{i}.bqkv", lw, "bqkv"), (f"layers.{i}.bo", lw, "bo"), (f"layers.{i}.b1", lw, "b1"),
                    (f"layers.{i}.b2", lw, "b2")]
    return out


def trainable_params(model: Model) -> dict[str, torch.Tensor]:
    """Named references to every trainable tensor (sf/model.py:234-249); BitFit's
    bq/bk/bv are views of the fused bias."""
    out = {}
    for name, owner, attr in _param_slots(model):
        t = getattr(owner, attr)
        if name.endswith(".bqkv"):
            i = name.split(".")[1]
            d = t.shape[0] // 3
            out[f"layers.{i}.bq"], out[f"layers.{i}.bk"], out[f"layers.{i}.bv"] = t[:d], t[d : 2 * d], t[2 * d :]
        else:
            out[name] = t
    if model.peft_method == "bitfit":  # reference order: bq, bk, bv, bo, b1, b2 per layer
        out = {k: out[k] for i in range(model.dims.n_layers) for k in (f"layers.{i}.{b}" for b in BIAS_NAMES)}
    return out


def make_peft_state(model: Model) -> PeftState:
    """Move every trainable tensor into one flat fp32 buffer (views keep the model
    pointing at the live parameters) and allocate float64 Adam moments."""
    slots = _param_slots(model)
    n = sum(getattr(o, a).numel() for _, o, a in slots)
    flat = torch.zeros(n, dtype=torch.float32, device=model.device)
    off = 0
    for _, owner, attr in slots:
        t = getattr(owner, attr)
        view = flat[off : off + t.numel()].view(t.shape)
        view.copy_(t)
        setattr(owner, attr, view)
        off += t.numel()
    st = PeftState(model.peft_method, trainable_params(model), flat,
                   torch.zeros(n, dtype=torch.float64, device=model.device), torch.zeros(n, dtype=torch.float64, device=model.device))
    return st


def backbone_param_count(model: Model) -> int:
    d = model.dims
    per = 4 * d.d_model * d.d_model + 4 * d.d_model + d.d_ff + d.d_model + 4 * d.d_model + 2 * d.d_model * d.d_ff
    return d.vocab * d.d_model + 2 * d.d_model + d.n_layers * per


def frozen_hash(model: Model) -> str:
    """SHA-256 over the frozen backbone bytes (sf/model.py:267-285, device byte layout)."""
    h = hashlib.sha256()
    skip = model.peft_method == "bitfit"
    for t in [model.weights.emb, model.weights.lnf_g, model.weights.lnf_b]:
        h.update(t.detach().cpu().contiguous().view(torch.uint8).numpy().tobytes())
    for lw in model.weights.layers:
        ts = [lw.wqkv, lw.wo, lw.ln1_g, lw.ln1_b, lw.ln2_g, lw.ln2_b, lw.mlp.w1_t, lw.mlp.w2]
        if not skip:
            ts += [lw.bqkv, lw.bo, lw.b1, lw.b2]
        for t in ts:
            h.update(t.detach().cpu().contiguous().view(torch.uint8).numpy().tobytes())
    return h.hexdigest()


# ---------------------------------------------------------------- LoRA packs


def _rp(r: int) -> int:
    return 8 if r <= 8 else 16


def ensure_lora_packs(model: Model) -> bool:
    """Build (once per parameter storage) the packed LoRA operands of every layer: rowproj packs
    (bf16 hi/lo [2][RP][K], lx_pack_params layout) of A_cat (q/k/v targets), each q/k/v B, A1, A2, B1, B2,
    and the K-extended q/k/v weight. Returns True when packs are live (refresh_lora_packs fills them).
    The fused q/k/v path needs equal ranks r % 8 == 0 with n * r <= 16 (cfg3: wq, wv at r = 8)."""
    if model.peft_method != "lora" or not model.lora:
        return False
    keys = sorted(model.lora)
    ptrs = tuple((model.lora[k].a.data_ptr(), model.lora[k].b.data_ptr()) for k in keys)
    st = model.__dict__.get("_lora_packs")
    if st is not None and st["ptrs"] == ptrs:
        return True
    if torch.cuda.is_available() and torch.cuda.is_current_stream_capturing():
        raise RuntimeError("ensure_lora_packs must run before CUDA-graph capture")
    dev, d = model.device, model.dims.d_model
    segs = []

    def seg(src: torch.Tensor, src_sr, src_sc, rows, cols, dst: torch.Tensor, dst_off, dst_sr, dst_sc, lo_off, scale=1.0):
        segs.append(_abi.PackSegment(src.data_ptr(), src_sr, src_sc, rows, cols, dst.data_ptr() + 2 * dst_off, dst_sr,
                                     dst_sc, lo_off, float(scale), 0))

    def pack_a(a: torch.Tensor, K: int):  # W(k, q) = A[k][q], A [K, r]
        r = a.shape[1]
        rp = _rp(r)
        t = torch.zeros(2, rp, K, dtype=torch.bfloat16, device=dev)
        seg(a, 1, r, r, K, t, 0, K, 1, rp * K)
        return t

    def pack_b(b: torch.Tensor, K: int):  # W(k, q) = B[q][k], B [r, K]
        r = b.shape[0]
        rp = _rp(r)
        t = torch.zeros(2, rp, K, dtype=torch.bfloat16, device=dev)
        seg(b, K, 1, r, K, t, 0, K, 1, rp * K)
        return t

    for i, lw in enumerate(model.weights.layers):
        lora = {t: model.lora[(i, t)] for t in model.lora_targets if (i, t) in model.lora}
        tq = tuple(t for t in ("wq", "wk", "wv") if t in lora)
        ranks = {lora[t].rank for t in tq}
        kx = 0
        if tq and len(ranks) == 1 and next(iter(ranks)) % 8 == 0 and len(tq) * next(iter(ranks)) <= 16:
            kx = len(tq) * next(iter(ranks))
        lp = {"kx": kx, "tq": tq, "b": {}}
        if kx:
            r = kx // len(tq)
            if lw.wqkv_ext is None or lw.wqkv_ext.shape != (d + kx, 3 * d + kx):
                ext = torch.zeros(d + kx, 3 * d + kx, dtype=torch.bfloat16, device=dev)
                ext[:d, : 3 * d] = lw.wqkv
                lw.wqkv_ext, lw.wqkv = ext, ext[:d, : 3 * d]
            ext, ld = lw.wqkv_ext, 3 * d + kx
            a_qkv = torch.zeros(2, kx, d, dtype=torch.bfloat16, device=dev)
            # the q/k/v B packs side by side ([n_t][2][RP][d]): equally spaced for the one-launch input-grad projection
            b_qkv = torch.zeros(len(tq), 2, _rp(r), d, dtype=torch.bfloat16, device=dev)
            lp["b_qkv"] = b_qkv
            for j, t in enumerate(tq):
                ad, sl = lora[t], QKV_SLOT[t]
                seg(ad.a, 1, r, r, d, a_qkv, j * r * d, d, 1, kx * d)  # rowproj pack rows j*r..
                seg(ad.b, d, 1, r, d, ext, (d + j * r) * ld + sl * d, ld, 1, 0, ad.scaling)  # s * B_j rows
                seg(ad.a, r, 1, d, r, ext, 3 * d + j * r, ld, 1, 0)  # A_j columns (input-grad GEMM)
                seg(ad.b, d, 1, r, d, b_qkv[j], 0, d, 1, _rp(r) * d)  # pack_b(ad.b, d) into slot j
                lp["b"][t] = b_qkv[j]
            lp["a_qkv"] = a_qkv
        if "w1" in lora and lora["w1"].rank <= 16:
            lp["a1"] = pack_a(lora["w1"].a, d)
            lp["b1"] = pack_b(lora["w1"].b, model.dims.d_ff)
        if "w2" in lora and lora["w2"].rank <= 16:
            lp["a2"] = pack_a(lora["w2"].a, model.dims.d_ff)
            lp["b2"] = pack_b(lora["w2"].b, d)
        lw.lora_pack = lp
    arr = (_abi.PackSegment * max(len(segs), 1))(*segs)
    host = torch.frombuffer(bytearray(bytes(arr)), dtype=torch.uint8)
    model.__dict__["_lora_packs"] = {"ptrs": ptrs, "segs": host.to(dev), "n": len(segs)}
    return True


def refresh_lora_packs(model: Model) -> None:
    """One launch: re-pack every LoRA factor after the optimizer step (stream-ordered, graph-capturable)."""
    st = model.__dict__.get("_lora_packs")
    if st is not None and st["n"]:
        _abi.call("lx_pack_params", st["segs"].data_ptr(), st["n"], _abi.stream_handle(model.device))


# ---------------------------------------------------------------- forward passes


def _items(x: torch.Tensor):
    """[s, d] or [B, s, d] -> (x2 [B*s, d], B, s)."""
    if x.dim() == 2:
        return x, 1, x.shape[0]
    return x.reshape(-1, x.shape[-1]), x.shape[0], x.shape[1]


def _mm_f32(a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    """bf16 x bf16 -> fp32 (cuBLAS)."""
    try:
        return torch.mm(a, b, out_dtype=torch.float32)
    except TypeError:  # older torch
        return torch.mm(a, b).float()


def lora_linear_forward(x, w, bias, adapter: LoraAdapter | None):
    """z = xW (+ bias) + scaling*(xA)B (sf/model.py:292-304); x bf16, z fp32."""
    if x.shape[1] != w.shape[0]:
        raise ShapeError(f"linear shapes disagree: {tuple(x.shape)} @ {tuple(w.shape)}")
    z = _mm_f32(x, w)
    cache = {"x": x, "ax": None}
    if adapter is not None:
        ax = x.float() @ adapter.a
        z.addmm_(ax, adapter.b, alpha=adapter.scaling)
        cache["ax"] = ax
    if bias is not None:
        z += bias
    return z, cache


class PendingResidual:
    """A block output whose residual add is deferred to the next LayerNorm: value = base + delta
    (fp32 base, bf16 delta [M, d]). The LN kernel materialises the fp32 sum it normalises."""

    __slots__ = ("base", "delta")

    def __init__(self, base: torch.Tensor, delta: torch.Tensor):
        self.base, self.delta = base, delta

    @property
    def shape(self):
        return self.base.shape

    def materialize(self) -> torch.Tensor:
        return (self.base.reshape(-1, self.base.shape[-1]) + self.delta.float()).view(self.base.shape)


def layernorm_forward(x, gamma, beta, eps: float = 1e-5, x_small_spec=None, delta=None, ext_cols: int = 0):
    """sf/model.py:307-312 on the fused kernel; x fp32 [M, d] -> bf16 y. x_small_spec=(s, m)
    additionally writes the predictor's downsampled rows (returned in the cache). With `delta`
    (bf16 [M, d]) -- or x a PendingResidual -- the residual add x + delta is fused: the fp32 sum
    is normalised and returned as cache["x"] (the block's y, sf/model.py:420)."""
    if isinstance(x, PendingResidual):
        x, delta = x.base, x.delta
    x2 = x.reshape(-1, x.shape[-1]).contiguous()
    M, d = x2.shape
    y_ext = torch.empty(M, d + ext_cols, dtype=torch.bfloat16, device=x2.device)  # + LoRA columns of a K-extended GEMM
    y = y_ext[:, :d] if ext_cols else y_ext
    mean = torch.empty(M, dtype=torch.float32, device=x2.device)
    istd = torch.empty(M, dtype=torch.float32, device=x2.device)
    resid = torch.empty(M, d, dtype=torch.float32, device=x2.device) if delta is not None else None
    xs, s, m = None, 0, 0
    if x_small_spec is not None:
        s, m = x_small_spec
        xs = torch.empty(M // s * m, d, dtype=torch.bfloat16, device=x2.device)
    _abi.call("lx_layernorm_fwd", x2.data_ptr(), _abi.ptr(delta), _abi.ptr(resid), M, d, gamma.data_ptr(), beta.data_ptr(),
              float(eps), y.data_ptr(), y_ext.stride(0), mean.data_ptr(), istd.data_ptr(), s, m, _abi.ptr(xs),
              _abi.stream_handle(x2.device))
    return y, {"x": resid if resid is not None else x2, "mean": mean, "inv_std": istd, "gamma": gamma, "x_small": xs,
               "y_ext": y_ext if ext_cols else None}


def adapter_forward(x: torch.Tensor, ad: AdapterLayer, resid: torch.Tensor | None = None):
    """x + relu(x Wd + bd) Wu + bu (sf/model.py:315-319) on the fp32 adapter kernel (csrc/adapter.cu); the cache
    keeps x, the pre-activation z and h = relu(z). With `resid` (fp32 [M, d]) the result is resid + adapter(x): the
    block's residual add (sf/model.py:420-427) fused into the kernel's store."""
    x = x.float().contiguous()
    M, d = x.shape
    r = ad.w_down.shape[1]
    z = torch.empty(M, r, dtype=torch.float32, device=x.device)
    out = torch.empty_like(x)
    rs = resid.reshape(M, d) if resid is not None else None
    if rs is not None and (rs.dtype != torch.float32 or rs.stride(1) != 1):
        raise ShapeError("adapter residual must be fp32 with unit column stride")
    _abi.call("lx_adapter_fwd", x.data_ptr(), d, M, d, r, ad.w_down.data_ptr(), ad.b_down.data_ptr(), ad.w_up.data_ptr(),
              ad.b_up.data_ptr(), z.data_ptr(), out.data_ptr(), d, _abi.ptr(rs), rs.stride(0) if rs is not None else 0,
              _abi.stream_handle(x.device))
    return out, {"x": x, "z": z, "h": torch.relu(z)}


def resolve_head_patterns(head_patterns, model_or_dpool, n_items: int, n_heads: int, device):
    """list[str] (shared) / list[list[str]] (per item) / int32 tensor [B|1, H] -> (pidx, item_stride)."""
    dp = model_or_dpool.dpool if isinstance(model_or_dpool, Model) else model_or_dpool
    if torch.is_tensor(head_patterns):
        t = head_patterns.to(device=device, dtype=torch.int32).contiguous()
        if t.dim() == 1:
            t = t[None]
        if t.shape[-1] != n_heads:
            raise ShapeError(f"expected {n_heads} head patterns, got {t.shape[-1]}")
        return t, (0 if t.shape[0] == 1 else n_heads)
    hp = list(head_patterns)
    if hp and isinstance(hp[0], (list, tuple)):
        rows = [[dp.idx(p) for p in row] for row in hp]
        if any(len(r) != n_heads for r in rows):
            raise ShapeError(f"expected {n_heads} head patterns per item")
        return torch.tensor(rows, dtype=torch.int32, device=device), n_heads
    if len(hp) != n_heads:
        raise ShapeError(f"expected {n_heads} head patterns, got {len(hp)}")
    # static assignments are lowered once per (assignment, device) and reused (also inside CUDA-graph capture)
    cache = dp.__dict__.setdefault("_static_idx", {})
    key = (tuple(str(p) for p in hp), str(device))
    if key not in cache:
        cache[key] = torch.tensor([[dp.idx(p) for p in hp]], dtype=torch.int32, device=device)
    return cache[key], 0


def linear(a: torch.Tensor, b_t: torch.Tensor, out_f32: bool = False, resid: torch.Tensor | None = None, bias=None,
           lora_x=None, lora_w=None, w_sr: int = 0, w_sc: int = 0, r: int = 0, scaling: float = 1.0, *,
           kn: bool = False, out: torch.Tensor | None = None) -> torch.Tensor:
    """out = (resid) + a @ b_t^T + bias + scaling * lora_x . w on the tcgen05 GEMM (fused epilogue).
    a bf16 [M, K] (any row stride), b_t bf16 [N, K] (K-major weight), or with kn=True the weight as
    stored for a @ W: [K, N] (any row stride). bias fp32 [N]. `out` (optional) receives the result."""
    M, K = a.shape
    N = b_t.shape[1] if kn else b_t.shape[0]
    if (b_t.shape[0] if kn else b_t.shape[1]) != K or b_t.stride(1) != 1 or a.stride(1) != 1:
        raise ShapeError(f"linear shapes disagree: {tuple(a.shape)} x {tuple(b_t.shape)} (kn={kn})")
    dt = torch.float32 if (out_f32 or resid is not None) else torch.bfloat16
    if out is None:
        out = torch.empty(M, N, dtype=dt, device=a.device)
    elif out.dtype != dt or tuple(out.shape) != (M, N) or out.stride(1) != 1:
        raise ShapeError(f"linear output {tuple(out.shape)} {out.dtype} does not match [{M}, {N}] {dt}")
    _abi.call("lx_linear_kn" if kn else "lx_linear", a.data_ptr(), a.stride(0), b_t.data_ptr(), b_t.stride(0), M, N, K,
              out.data_ptr(), out.stride(0), int(out.dtype == torch.float32), _abi.ptr(resid), _abi.ptr(bias),
              _abi.ptr(lora_x), _abi.ptr(lora_w), w_sr, w_sc, r if lora_x is not None else 0, float(scaling),
              _abi.stream_handle(a.device))
    return out


QKV_SLOT = {"wq": 0, "wk": 1, "wv": 2}
# LX_NO_PACK=1: MLP GEMMs gather the active neuron blocks straight from W (one TMA box per block)
# instead of streaming item-packed copies (experiments)
_NO_PACK = __import__("os").environ.get("LX_NO_PACK", "0") == "1"
_PACK_CACHE_BYTES = float(__import__("os").environ.get("LX_PACK_CACHE_GB", "48")) * 2**30


# LX_SIDE_ROWPROJ=0: the LoRA down-projections of the LN outputs (x A_qkv, h2 A1) on the main stream instead of an
# auxiliary stream beside the attention-predictor / MLP-mask chains they do not depend on
_SIDE_ROWPROJ = __import__("os").environ.get("LX_SIDE_ROWPROJ", "1") != "0"
_AUX_STREAMS: dict = {}


def _aux_stream(device):
    if not _SIDE_ROWPROJ:
        return None
    key = torch.device(device).index
    if key not in _AUX_STREAMS:
        _AUX_STREAMS[key] = torch.cuda.Stream(device=device)
    return _AUX_STREAMS[key]


def _side_call(fn, inputs, device):
    """Run fn() on the auxiliary stream after everything queued so far; returns a handle for _side_join. Inputs
    made on the main stream are recorded on the side stream (allocator safety); captured into a CUDA graph as a
    fork / join like the engine's other side stream."""
    side = _aux_stream(device)
    if side is None:
        return (fn(), None)
    main = torch.cuda.current_stream(device)
    side.wait_stream(main)
    with torch.cuda.stream(side):
        out = fn()
    for t in inputs:
        t.record_stream(side)
    return (out, side)


def _side_join(handle):
    """The result of a _side_call, with the main stream ordered after it."""
    out, side = handle
    if side is not None:
        main = torch.cuda.current_stream(out.device)
        main.wait_stream(side)
        out.record_stream(main)
    return out


def _qkv_ext_ready(lw, lora: dict, x_ext) -> bool:
    """The q/k/v LoRA rides in the projection GEMM by K-extension (mha_forward's ext path)."""
    tq = [t for t in ("wq", "wk", "wv") if t in lora]
    lp = lw.lora_pack
    return bool(tq) and x_ext is not None and lp is not None and lp["kx"] > 0 and lp["tq"] == tuple(tq)


def _qkv_lora(lora: dict, d: int):
    """Targets among wq/wk/wv and their concatenated A [d, n*r] (sf/model.py:292-304): one rowproj
    computes x A for all of them."""
    tq = [t for t in ("wq", "wk", "wv") if t in lora]
    if not tq:
        return tq, None, 0
    r = lora[tq[0]].rank
    a_cat = lora[tq[0]].a if len(tq) == 1 else torch.cat([lora[t].a for t in tq], 1).contiguous()
    return tq, a_cat, r


# The dense projections are plain library GEMMs (bias in the cuBLAS addmm). LX_PROJ_ENGINE=1 runs them on the
# tcgen05 engine instead (lx_linear_kn / lx_linear, fp32 bias in the epilogue): measured 13% slower per GEMM inside
# the cfg3 step (56.9 vs 49.7 us forward, 52.0 vs 46.0 us input-grad; +0.6 ms per step), so not default.
_PROJ_CUBLAS = __import__("os").environ.get("LX_PROJ_ENGINE", "0") != "1"


def _proj(a: torch.Tensor, w: torch.Tensor, bias: torch.Tensor, bias16=None) -> torch.Tensor:
    """bf16 a @ w + bias for a projection weight stored [K, N] (sf/model.py:340-354): cuBLAS addmm with the bf16
    bias, or (LX_PROJ_ENGINE=1) the tcgen05 engine with the fp32 bias in the epilogue (lx_linear_kn)."""
    if _PROJ_CUBLAS:
        return torch.addmm(bias16, a, w)
    return linear(a, w, bias=bias, kn=True)


def proj_t(a: torch.Tensor, w: torch.Tensor) -> torch.Tensor:
    """bf16 a @ w^T for a projection weight stored [N, K] row-major (the input-grads dx = dy W^T,
    sf/autograd.py:127-162): cuBLAS, or (LX_PROJ_ENGINE=1) lx_linear with w as the K-major operand."""
    if _PROJ_CUBLAS:
        return torch.mm(a, w.t())
    return linear(a, w)


def _bias_bf16(lw: LayerWeights, name: str, frozen: bool) -> torch.Tensor:
    """bf16 copy of a projection bias for the cuBLAS addmm; frozen biases (every PEFT method but BitFit)
    are converted once per storage instead of once per step."""
    src = getattr(lw, name)
    if not frozen:
        return src.to(torch.bfloat16)
    cache = lw.__dict__.setdefault("_bias_bf16", {})
    key = (name, src.data_ptr())
    if key not in cache:
        cache[key] = src.to(torch.bfloat16)
    return cache[key]


def mha_forward(x, lw: LayerWeights, lora: dict, head_patterns, pool, dims: ModelDims, counter=None, *, dpool=None,
                x_ext=None, frozen_bias: bool = False, ax_pre=None):
    """Block-sparse multi-head attention (sf/model.py:322-360). x: LN1 output bf16 [B, s, d] (or [s, d]).
    The dense projections are plain library GEMMs (_proj: cuBLAS, bias in the addmm); the q/k/v LoRA deltas
    ride in the same GEMM by K-extension ([x | xA] x [W ; s B]), else each is a rank-r update of its column slice.
    Returns (out bf16 [B*s, d] = O Wo + bo (+ LoRA), cache); the cache holds O and the row LSE
    instead of probabilities. The residual add is fused into the next LayerNorm kernel."""
    x2, B, s = _items(x)
    d, H, hd = dims.d_model, dims.n_heads, dims.head_dim
    dp = dpool if dpool is not None else device_pool(pool, x2.device, dims.seq_len, dims.attn_blk)
    pidx, stride = resolve_head_patterns(head_patterns, dp, B, H, x2.device)
    tq = [t for t in ("wq", "wk", "wv") if t in lora]
    lp = lw.lora_pack
    ext = _qkv_ext_ready(lw, lora, x_ext)
    # the concatenated A is only an operand of the unfused path (the fused one reads the packs)
    tq, a_cat, r = _qkv_lora(lora, d) if not ext else (tq, None, lora[tq[0]].rank)
    bqkv16 = _bias_bf16(lw, "bqkv", frozen_bias) if _PROJ_CUBLAS else None
    ax = None
    if ext:
        # K-extended projection: x_ext = [x | xA_cat] (bf16 LoRA columns written by the rowproj), W_ext rows d.. = s*B
        kx = lp["kx"]
        if ax_pre is not None:  # launched on the auxiliary stream right after LN1 (block_forward)
            ax = _side_join(ax_pre)
        else:
            ax = rowproj_packed(x_ext, B, s, d, lp["a_qkv"], kx, out_bf16=x_ext[:, d:])  # fp32 [M, n*r] for the grads
        qkv = _proj(x_ext, lw.wqkv_ext[: d + kx, : 3 * d], lw.bqkv, bqkv16)
    else:
        qkv = _proj(x2, lw.wqkv, lw.bqkv, bqkv16)  # bf16 [M, 3d]
    if tq and not ext:
        ax = rowproj(x2, B, s, d, a_cat, a_cat.shape[1], 1, a_cat.shape[1])  # fp32 [M, n*r] (kept for the LoRA grads)
        axb = ax.to(torch.bfloat16)
        for j, t in enumerate(tq):
            sl = QKV_SLOT[t]
            qkv[:, sl * d : (sl + 1) * d].addmm_(axb[:, j * r : (j + 1) * r], (lora[t].b * lora[t].scaling).to(torch.bfloat16))
    scale = 1.0 / float(np.sqrt(hd))
    o, lse = attention_forward(qkv[:, :d], qkv[:, d : 2 * d], qkv[:, 2 * d :], 3 * d, B, s, H, hd, pidx, stride, dp, scale)
    if counter is not None:
        nnz = sum(dp_nnz(dp, int(i)) for i in pidx.flatten().tolist()) * (B if stride == 0 else 1)
        counter.add(2 * nnz * dims.attn_blk * dims.attn_blk * hd)
    out = _proj(o, lw.wo, lw.bo, _bias_bf16(lw, "bo", frozen_bias) if _PROJ_CUBLAS else None)  # bf16 [M, d]
    ad_o = lora.get("wo")
    ax_o = None
    if ad_o is not None:
        ax_o = rowproj(o, B, s, d, ad_o.a, ad_o.rank, 1, ad_o.rank)
        out.addmm_(ax_o.to(torch.bfloat16), (ad_o.b * ad_o.scaling).to(torch.bfloat16))
    cache = {"x": x2, "qkv": qkv, "o": o, "lse": lse, "pidx": pidx, "stride": stride, "ax": ax, "lora_t": tq,
             "lora_r": r, "a_cat": a_cat, "ax_o": ax_o, "n_items": B, "s": s, "dpool": dp, "ext": ext}
    return out, cache


def dp_nnz(dp: DevicePool, i: int) -> int:
    n_b = dp.seq_len // dp.attn_blk
    return len(build_pool(n_b)[dp.ids[i]].coords) if dp.seq_len else 0


def mlp_forward(x, lw: LayerWeights, lora: dict, neuron_mask, dims: ModelDims, counter=None, *, resid=None,
                out_f32: bool = False, ax1_pre=None):
    """ReLU MLP restricted to active neuron blocks (sf/model.py:363-400) on the tcgen05
    gather-GEMMs with bias / LoRA / ReLU fused in the epilogues. x: LN2 output bf16.
    With `resid` (fp32) the fc2 epilogue returns resid + MLP (the block's residual add)."""
    x2, B, s = _items(x)
    d, f, blk = dims.d_model, dims.d_ff, dims.blk_size
    nm = lower_mask(neuron_mask, dims.n_blk, blk, B, x2.device)
    ad1, ad2 = lora.get("w1"), lora.get("w2")
    # active rows of W1^T and W2 packed per item once per layer; kept for the backward's input-grads unless the
    # packs of all layers would exceed LX_PACK_CACHE_GB (capacity [B, d_ff, d] per weight: 137 GB at OPT-6.7B,
    # B = 16), in which case the backward re-packs its layer (mlp_backward)
    pack = not _NO_PACK
    w1p, w2p = neuron_ops.pack_active_rows2(lw.mlp.w1_t, lw.mlp.w2, nm) if pack else (None, None)
    keep = pack and dims.n_layers * 2 * B * f * d * 2 <= _PACK_CACHE_BYTES
    lp = lw.lora_pack
    if ad1 is None:
        ax1 = None
    elif ax1_pre is not None:  # launched on the auxiliary stream right after LN2 (block_forward)
        ax1 = _side_join(ax1_pre)
    elif lp is not None and lp.get("a1") is not None:
        ax1 = rowproj_packed(x2, B, s, d, lp["a1"], ad1.rank)
    else:
        ax1 = rowproj(x2, B, s, d, ad1.a, ad1.rank, 1, ad1.rank)
    # relu'(z) as bits beside the bf16 activation: the fc2 input-grad epilogue reads 1/16 of the bytes
    relu_bits = torch.empty(B * s, f // 16, dtype=torch.int16, device=x2.device) if f % 16 == 0 else None
    hid = neuron_ops.neuron_matmul_fwd1(x2.view(B, s, d), lw.mlp, nm, blk, counter, bias=lw.b1, ax=ax1,
                                        lora_b=ad1.b if ad1 else None, lora_r=ad1.rank if ad1 else 0,
                                        scaling=ad1.scaling if ad1 else 1.0, relu=True, w_packed=w1p,
                                        relu_bits=relu_bits)
    if ad2 is None:
        ax2 = None
    elif lp is not None and lp.get("a2") is not None:
        ax2 = rowproj_packed(hid.values, B, s, f, lp["a2"], ad2.rank, masks=nm, blk=blk)
    else:
        ax2 = rowproj(hid.values, B, s, f, ad2.a, ad2.rank, 1, ad2.rank, masks=nm, blk=blk)
    out = neuron_ops.neuron_matmul_fwd2(
        hid, lw.mlp, None, counter, bias=lw.b2, ax=ax2, lora_b=ad2.b if ad2 else None, lora_r=ad2.rank if ad2 else 0,
        scaling=ad2.scaling if ad2 else 1.0, resid=resid, w_packed=w2p,
        out=torch.empty(B * s, d, dtype=torch.float32, device=x2.device) if (out_f32 or resid is not None) else None)
    if counter is not None:
        n_act = int(nm.counts.sum()) * blk
        if ad1 is not None:
            counter.add(s * (d + n_act // max(B, 1)) * ad1.rank * B)
        if ad2 is not None:
            counter.add(s * (n_act // max(B, 1) + d) * ad2.rank * B)
    return out, {"x": x2, "a": hid, "mask": nm, "ax1": ax1, "ax2": ax2, "n_items": B, "s": s, "relu_bits": relu_bits,
                 "w1p": w1p if keep else None, "w2p": w2p if keep else None, "repack": pack and not keep}


def block_forward(x, model: Model, layer: int, masks, counter=None):
    """Pre-norm residual block (sf/model.py:403-433); x fp32 [B, s, d]. `masks` is a
    LayerMasks or a provider with attn_patterns(layer, h) / mlp_mask(layer, h)."""
    lw = model.weights.layers[layer]
    lora = {t: model.lora[(layer, t)] for t in model.lora_targets} if model.peft_method == "lora" else {}
    B, s, d = x.shape  # x: fp32 [B, s, d] or a PendingResidual (previous block's y + MLP)
    static = isinstance(masks, LayerMasks)
    spec = None
    if not static and getattr(masks, "fused_downsample", False):
        from .predictor import downsample_indices

        spec = (s, len(downsample_indices(s)))
    kx = lw.lora_pack["kx"] if (model.peft_method == "lora" and lw.lora_pack is not None) else 0
    h1, c1 = layernorm_forward(x, lw.ln1_g, lw.ln1_b, x_small_spec=spec, ext_cols=kx)
    h1v = h1.view(B, s, d)
    # the q/k/v LoRA down-projection x A_qkv only needs LN1's output: it runs beside the attention predictor
    ax_pre = None
    if not static and _qkv_ext_ready(lw, lora, c1["y_ext"]):
        ye, lp = c1["y_ext"], lw.lora_pack
        ax_pre = _side_call(lambda: rowproj_packed(ye, B, s, d, lp["a_qkv"], lp["kx"], out_bf16=ye[:, d:]), [ye], h1.device)
    if static:
        hp = masks.head_patterns
    elif spec is not None:
        hp = masks.attn_patterns(layer, h1v, x_small=c1["x_small"])
    else:
        hp = masks.attn_patterns(layer, h1v)
    adapter = model.peft_method == "adapter"
    x2 = c1["x"]  # the block input (materialised by LN1 when x was a pending residual)
    att, ca = mha_forward(h1v, lw, lora, hp, model.pool, model.dims, counter, dpool=model.dpool, x_ext=c1["y_ext"],
                          frozen_bias=model.peft_method != "bitfit", ax_pre=ax_pre)
    caa = None
    if adapter:
        # y = x + adapter(attn): the residual add fused into the adapter kernel's store
        y_att, caa = adapter_forward(att, model.adapters[(layer, "attn")], resid=x2)
        h2, c2 = layernorm_forward(y_att.view(B, s, d), lw.ln2_g, lw.ln2_b)
    else:
        # y = x + attn fused into the LN2 kernel (fp32 y returned as the LN cache input)
        h2, c2 = layernorm_forward(x2, lw.ln2_g, lw.ln2_b, delta=att)
    y = c2["x"]
    h2v = h2.view(B, s, d)
    # the w1 LoRA down-projection h2 A1 only needs LN2's output: it runs beside the MLP-mask prediction
    ax1_pre = None
    lp = lw.lora_pack
    if not static and "w1" in lora and lp is not None and lp.get("a1") is not None:
        r1 = lora["w1"].rank
        ax1_pre = _side_call(lambda: rowproj_packed(h2, B, s, d, lp["a1"], r1), [h2], h1.device)
    nm = masks.neuron_mask if static else masks.mlp_mask(layer, h2v)
    # the MLP's residual add (y + MLP) is deferred into the next LayerNorm: fc2 stores bf16 only
    mo, cm = mlp_forward(h2v, lw, lora, nm, model.dims, counter, out_f32=adapter, ax1_pre=ax1_pre)
    cma = None
    if adapter:
        out, cma = adapter_forward(mo, model.adapters[(layer, "mlp")], resid=y)
        out = out.view(B, s, d)
    else:
        out = PendingResidual(y.view(B, s, d), mo)
    cache = {"ln1": c1, "attn": ca, "attn_adapter": caa, "ln2": c2, "mlp": cm, "mlp_adapter": cma,
             "masks": LayerMasks(ca["pidx"], cm["mask"])}
    return out, cache


def model_forward(model: Model, tokens, masks, counter=None):
    """Embed, run all blocks, final LN, tied unembedding (sf/model.py:436-451).
    tokens [s] or [B, s]; returns fp32 logits of the same leading shape."""
    tok = torch.as_tensor(np.asarray(tokens) if not torch.is_tensor(tokens) else tokens).to(model.device, torch.int64)
    squeeze = tok.dim() == 1
    if squeeze:
        tok = tok[None]
    if int(tok.max()) >= model.dims.vocab or int(tok.min()) < 0:
        raise ValueError("token id out of vocab range")
    B, s = tok.shape
    if ensure_lora_packs(model):
        refresh_lora_packs(model)
    h = torch.nn.functional.embedding(tok, model.weights.emb).float()
    caches = []
    for layer in range(model.dims.n_layers):
        lm = masks[layer] if isinstance(masks, list) else masks
        h, c = block_forward(h, model, layer, lm, counter)
        caches.append(c)
    hf, cf = layernorm_forward(h, model.weights.lnf_g, model.weights.lnf_b)
    logits = _mm_f32(hf, model.weights.emb.t())
    logits = logits.view(s, -1) if squeeze else logits.view(B, s, -1)
    return logits, {"blocks": caches, "lnf": cf, "hf": hf, "tokens": tok}


def loss_forward(logits, targets) -> float:
    """Mean cross-entropy over positions (sf/model.py:454-462); batched input averages items."""
    t = torch.as_tensor(np.asarray(targets) if not torch.is_tensor(targets) else targets).to(logits.device, torch.int64)
    V = logits.shape[-1]
    if int(t.max()) >= V or int(t.min()) < 0:
        raise ValueError("target id out of vocab range")
    return float(torch.nn.functional.cross_entropy(logits.reshape(-1, V).float(), t.reshape(-1)))


def loss_backward(logits, targets) -> torch.Tensor:
    """d loss / d logits (sf/model.py:465-472): per item (softmax - onehot) / s."""
    t = torch.as_tensor(np.asarray(targets) if not torch.is_tensor(targets) else targets).to(logits.device, torch.int64)
    V = logits.shape[-1]
    g = torch.softmax(logits.reshape(-1, V).float(), dim=-1)
    g[torch.arange(g.shape[0], device=g.device), t.reshape(-1)] -= 1.0
    return (g / t.shape[-1]).view(logits.shape)
