"""Neuron-centric sparse MLP on the B200 (drop-in for sf/neuron_ops.py).

Device layout (sf/neuron_ops.py:1-8): W1 is kept as W1^T
[d_ff, d] and W2 as [d_ff, d], both bf16 row-major, so every neuron block is
`blk` contiguous rows that one TMA box streams. A neuron mask is lowered once
per layer to device index lists (`NeuronMasks`: counts, ascending ids, inverse
positions) that the tcgen05 gather-GEMMs consume; hidden activations are
packed per item (`ActiveHidden`), exactly the reference's packed order.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _abi
from .errors import MaskError, ShapeError


def block_slices(d_ff: int, blk_size: int) -> list[slice]:
    """sf/neuron_ops.py:22-24."""
    return [slice(lo, min(lo + blk_size, d_ff)) for lo in range(0, d_ff, blk_size)]


def n_blocks(d_ff: int, blk_size: int) -> int:
    """sf/neuron_ops.py:27-28."""
    return (d_ff + blk_size - 1) // blk_size


@dataclass
class LayeredWeights:
    """W1 (logically d x d_ff, stored as W1^T) and W2 (d_ff x d), bf16 on device (sf/neuron_ops.py:31-45)."""

    w1_t: torch.Tensor  # [d_ff, d]
    w2: torch.Tensor  # [d_ff, d]
    layout_w1: str = "col"
    layout_w2: str = "row"

    @classmethod
    def from_row_major(cls, w1, w2, device=None) -> "LayeredWeights":
        w1 = torch.as_tensor(np.asarray(w1) if not torch.is_tensor(w1) else w1)
        w2 = torch.as_tensor(np.asarray(w2) if not torch.is_tensor(w2) else w2)
        dev = device or "cuda"
        return cls(w1.t().contiguous().to(dev, torch.bfloat16), w2.contiguous().to(dev, torch.bfloat16))

    @property
    def w1(self) -> torch.Tensor:
        return self.w1_t.t()

    def to_row_major(self):
        return self.w1_t.t().contiguous(), self.w2


@dataclass
class NeuronMasks:
    """Device form of per-item neuron-block masks (sf/predictor.py:128-139 output, lowered)."""

    counts: torch.Tensor  # int32 [B]
    ids: torch.Tensor  # int32 [B, n_blk] ascending active block ids (first counts[b] valid)
    pos: torch.Tensor  # int32 [B, n_blk] packed position or -1
    n_blk: int
    blk: int

    @property
    def n_items(self) -> int:
        return self.counts.shape[0]

    def to_bool(self) -> torch.Tensor:
        """[B, n_blk] bool (host-typed view for parity / reference API)."""
        return self.pos >= 0

    def expand(self, n_items: int) -> "NeuronMasks":
        if self.n_items == n_items:
            return self
        if self.n_items != 1:
            raise MaskError(f"mask for {self.n_items} items used with {n_items}")
        return NeuronMasks(self.counts.expand(n_items).contiguous(), self.ids.expand(n_items, -1).contiguous(),
                           self.pos.expand(n_items, -1).contiguous(), self.n_blk, self.blk)


_HOST_MASK_CACHE: dict = {}


def _pack_bits(mask_bool: torch.Tensor) -> torch.Tensor:
    B, n = mask_bool.shape
    words = (n + 31) // 32
    m = torch.zeros(B, words * 32, dtype=torch.int64, device=mask_bool.device)
    m[:, :n] = mask_bool.to(torch.int64)
    w = (m.view(B, words, 32) << torch.arange(32, device=mask_bool.device, dtype=torch.int64)).sum(-1)
    w = torch.where(w >= 2**31, w - 2**32, w)
    return w.to(torch.int32).contiguous()


def lower_mask(mask, n_blk: int, blk: int, n_items: int | None = None, device=None) -> NeuronMasks:
    """bool [n_blk] (shared) or [B, n_blk] (per item) -> NeuronMasks (device compaction, no host sync)."""
    if isinstance(mask, NeuronMasks):
        if mask.n_blk != n_blk:
            raise MaskError(f"mask length {mask.n_blk} != n_blk {n_blk}")
        return mask.expand(n_items) if n_items else mask
    if not torch.is_tensor(mask):
        # host masks (static LayerMasks / reference-typed providers) are lowered once and reused,
        # which also keeps host->device copies out of CUDA-graph capture
        arr = np.ascontiguousarray(np.asarray(mask, dtype=bool))
        key = (arr.tobytes(), arr.shape, n_blk, blk, n_items, str(device or "cuda"))
        hit = _HOST_MASK_CACHE.get(key)
        if hit is None:
            hit = lower_mask(torch.from_numpy(arr).to(device or "cuda"), n_blk, blk, n_items, device)
            if len(_HOST_MASK_CACHE) > 256:
                _HOST_MASK_CACHE.clear()
            _HOST_MASK_CACHE[key] = hit
        return hit
    t = mask.to(device or "cuda", torch.bool)
    if t.dim() == 1:
        t = t[None]
    if t.shape[-1] != n_blk:
        raise MaskError(f"mask length ({t.shape[-1]},) != n_blk ({n_blk},)")
    if n_items and t.shape[0] == 1 and n_items > 1:
        t = t.expand(n_items, n_blk)
    B = t.shape[0]
    bits = _pack_bits(t)
    counts = torch.empty(B, dtype=torch.int32, device=t.device)
    ids = torch.zeros(B, n_blk, dtype=torch.int32, device=t.device)
    pos = torch.empty(B, n_blk, dtype=torch.int32, device=t.device)
    _abi.call("lx_mask_compact", bits.data_ptr(), B, n_blk, 0, counts.data_ptr(), ids.data_ptr(), pos.data_ptr(),
              _abi.stream_handle(t.device))
    return NeuronMasks(counts, ids, pos, n_blk, blk)


@dataclass
class ActiveHidden:
    """Packed active hidden columns (sf/neuron_ops.py:48-56), per item: row t of item b holds
    its first counts[b]*blk columns in ascending block order."""

    values: torch.Tensor  # bf16 [B*s, d_ff] (row stride d_ff; only the packed prefix is valid)
    masks: NeuronMasks
    blk_size: int
    d_ff: int
    n_items: int = 1

    def packed(self, item: int = 0) -> torch.Tensor:
        """Host-typed [s, F_act] view of one item (syncs)."""
        s = self.values.shape[0] // self.n_items
        f = int(self.masks.counts[item]) * self.blk_size
        return self.values[item * s : (item + 1) * s, :f]

    @property
    def active_blocks(self) -> tuple[int, ...]:
        c = int(self.masks.counts[0])
        return tuple(int(b) for b in self.masks.ids[0, :c].tolist())

    @property
    def col_index(self) -> np.ndarray:
        return np.concatenate([np.arange(b * self.blk_size, min((b + 1) * self.blk_size, self.d_ff)) for b in self.active_blocks]) \
            if self.active_blocks else np.empty(0, dtype=int)


def active_columns(mask, d_ff: int, blk_size: int) -> tuple[tuple[int, ...], np.ndarray]:
    """sf/neuron_ops.py:59-72 (host-typed helper)."""
    m = mask.detach().cpu().numpy() if torch.is_tensor(mask) else np.asarray(mask, dtype=bool)
    m = m.astype(bool)
    if m.shape != (n_blocks(d_ff, blk_size),):
        raise MaskError(f"mask length {m.shape} != n_blk ({n_blocks(d_ff, blk_size)},)")
    active = tuple(int(b) for b in np.flatnonzero(m))
    sl = block_slices(d_ff, blk_size)
    cols = np.concatenate([np.arange(sl[b].start, sl[b].stop) for b in active]) if active else np.empty(0, dtype=int)
    return active, cols


def _as_items(x: torch.Tensor) -> tuple[torch.Tensor, int, int]:
    if x.dim() == 2:
        return x.contiguous(), 1, x.shape[0]
    B, s, d = x.shape
    return x.reshape(B * s, d).contiguous(), B, s


def _check_device_blk(d_ff: int, blk: int) -> None:
    if d_ff % blk:
        raise MaskError(f"d_ff {d_ff} must be a multiple of blk_size {blk} on the sm_100a path (ragged tail unsupported)")


def neuron_matmul_fwd1(x, weights: LayeredWeights, mask, blk_size: int, counter=None, *, bias=None, ax=None, lora_b=None,
                       lora_r=0, scaling=1.0, relu=False, out=None, w_packed=None, relu_bits=None) -> ActiveHidden:
    """x @ W1[:, cols] over active column blocks (sf/neuron_ops.py:75-82) on the tcgen05
    N-gather GEMM. Optional fused epilogue (used by mlp_forward): + bias[cols] + scaling*ax B[:,cols], ReLU.
    `relu_bits` (int16 [M, d_ff/16], with relu): also receives relu'(z) as bits for lx_neuron_fc2_dgrad."""
    d_ff, d = weights.w1_t.shape
    _check_device_blk(d_ff, blk_size)
    x2, B, s = _as_items(x.to(torch.bfloat16))
    nm = lower_mask(mask, n_blocks(d_ff, blk_size), blk_size, B, x2.device)
    vals = out if out is not None else torch.empty(B * s, d_ff, dtype=torch.bfloat16, device=x2.device)
    _abi.call("lx_neuron_fc1", x2.data_ptr(), B, s, d, d_ff, blk_size, weights.w1_t.data_ptr(), nm.counts.data_ptr(),
              nm.ids.data_ptr(), _abi.ptr(bias), _abi.ptr(ax), _abi.ptr(lora_b), lora_r, float(scaling), int(relu),
              vals.data_ptr(), d_ff, _abi.ptr(w_packed), _abi.ptr(relu_bits), _abi.stream_handle(x2.device))
    if counter is not None:
        counter.add(s * d * int(nm.counts.sum()) * blk_size)
    return ActiveHidden(vals, nm, blk_size, d_ff, B)


def neuron_matmul_fwd2(hidden: ActiveHidden, weights: LayeredWeights, mask, counter=None, *, bias=None, ax=None,
                       lora_b=None, lora_r=0, scaling=1.0, out=None, resid=None, w_packed=None) -> torch.Tensor:
    """Packed hidden @ W2[cols, :] (sf/neuron_ops.py:85-95) on the tcgen05 K-gather GEMM.
    With `resid` (fp32 [M, d]) the result is fp32 resid + MLP (fused residual add)."""
    d_ff, d = weights.w2.shape
    nm = hidden.masks
    if mask is not None and mask is not nm:
        other = lower_mask(mask, nm.n_blk, hidden.blk_size, nm.n_items, hidden.values.device)
        if not torch.equal(other.pos, nm.pos):
            raise MaskError("mask does not match the mask the hidden activations were computed with")
    M = hidden.values.shape[0]
    s = M // hidden.n_items
    f32 = resid is not None
    res = out if out is not None else torch.empty(M, d, dtype=torch.float32 if f32 else torch.bfloat16,
                                                  device=hidden.values.device)
    _abi.call("lx_neuron_fc2", hidden.values.data_ptr(), hidden.values.stride(0), hidden.n_items, s, d, d_ff,
              hidden.blk_size, weights.w2.data_ptr(), nm.counts.data_ptr(), nm.ids.data_ptr(), _abi.ptr(bias),
              _abi.ptr(ax), _abi.ptr(lora_b), lora_r, float(scaling), res.data_ptr(), int(res.dtype == torch.float32),
              _abi.ptr(resid), _abi.ptr(w_packed), _abi.stream_handle(res.device))
    if counter is not None:
        counter.add(s * int(nm.counts.sum()) * hidden.blk_size * d)
    return res


def pack_active_rows2(w_a: torch.Tensor, w_b: torch.Tensor, masks: NeuronMasks) -> tuple[torch.Tensor, torch.Tensor]:
    """pack_active_rows of two [d_ff, d] weights under the same masks (W1^T and W2 of a layer) in one launch."""
    d_ff, d = w_a.shape
    if tuple(w_b.shape) != (d_ff, d) or w_b.dtype != w_a.dtype:
        raise ShapeError("pack_active_rows2: the two weights must have the same shape and dtype")
    pa = torch.empty(masks.n_items, d_ff, d, dtype=w_a.dtype, device=w_a.device)
    pb = torch.empty_like(pa)
    _abi.call("lx_pack_active_rows2", w_a.data_ptr(), w_b.data_ptr(), d_ff, d, masks.blk, masks.n_items,
              masks.counts.data_ptr(), masks.ids.data_ptr(), pa.data_ptr(), pb.data_ptr(), _abi.stream_handle(w_a.device))
    return pa, pb


def pack_active_rows(w: torch.Tensor, masks: NeuronMasks) -> torch.Tensor:
    """Item-packed copy [B, d_ff, d] of a [d_ff, d] weight's active block rows (ascending), so the
    tcgen05 GEMMs stream them with large TMA boxes (csrc/abi_gemm.cu lx_pack_active_rows)."""
    d_ff, d = w.shape
    out = torch.empty(masks.n_items, d_ff, d, dtype=w.dtype, device=w.device)
    _abi.call("lx_pack_active_rows", w.data_ptr(), d_ff, d, masks.blk, masks.n_items, masks.counts.data_ptr(),
              masks.ids.data_ptr(), out.data_ptr(), _abi.stream_handle(w.device))
    return out


# ---------------------------------------------------------------- skinny LoRA helpers (csrc/lora.cu)


def rowproj(x2: torch.Tensor, n_items: int, s: int, K: int, w: torch.Tensor, w_sk: int, w_sq: int, r: int,
            scale: float = 1.0, masks: NeuronMasks | None = None, blk: int = 1, out: torch.Tensor | None = None) -> torch.Tensor:
    """Y[M, r] = scale * X[M, K] W (K gathered per item when `masks` is given). `out` may be a column
    slice of a wider fp32 buffer (row stride out.stride(0))."""
    y = out if out is not None else torch.empty(x2.shape[0], r, dtype=torch.float32, device=x2.device)
    nbytes = int(_abi.lib().lx_rowproj_ws_bytes(n_items, K, r, int(masks is not None)))
    ws = torch.empty(nbytes, dtype=torch.uint8, device=x2.device)
    _abi.call("lx_rowproj", x2.data_ptr(), x2.stride(0), n_items, s, K, w.data_ptr(), w_sk, w_sq, r, float(scale),
              _abi.ptr(masks.counts if masks else None), _abi.ptr(masks.ids if masks else None), blk, y.data_ptr(),
              y.stride(0), ws.data_ptr(), _abi.stream_handle(x2.device))
    return y


def rowproj_packed(x2: torch.Tensor, n_items: int, s: int, K: int, wpack: torch.Tensor, r: int, scale: float = 1.0,
                   masks: NeuronMasks | None = None, blk: int = 1, out: torch.Tensor | None = None,
                   out_bf16: torch.Tensor | None = None) -> torch.Tensor:
    """Y[M, r] = scale * X[M, K] W over a pre-packed W (lx_pack_params layout [2][RP][K_full], hi then lo);
    K gathered per item through `masks` (packed k -> ids[b][k/blk]*blk + k%blk of the full pack).
    `out_bf16` (optional, row-strided) receives a bf16 copy of Y."""
    y = out if out is not None else torch.empty(x2.shape[0], r, dtype=torch.float32, device=x2.device)
    _abi.call("lx_rowproj_packed", x2.data_ptr(), x2.stride(0), n_items, s, K, wpack.data_ptr(), wpack.shape[2],
              wpack.shape[1], r, float(scale), _abi.ptr(masks.counts if masks else None),
              _abi.ptr(masks.ids if masks else None), blk, y.data_ptr(), y.stride(0), _abi.ptr(out_bf16),
              out_bf16.stride(0) if out_bf16 is not None else 0, _abi.stream_handle(x2.device))
    return y


ROWPROJ_SEG_MAX_K = 4096  # lx_rowproj_packed_seg stages X rows in shared memory (kRpsMaxK in csrc/lora.cu)


def rowproj_packed_seg(x2: torch.Tensor, x_seg: int, K: int, wpacks: torch.Tensor, r: int, scale: float, y: torch.Tensor,
                       y_seg: int, yb: torch.Tensor | None, yb_seg: int, n_seg: int) -> None:
    """n_seg dense rowproj_packed problems in one launch: Y_k = scale * X_k W_k with X_k = x2 columns offset by
    k * x_seg, W_k = wpacks[k] ([n_seg][2][RP][K_full]), Y_k / yb_k at column offsets k * y_seg / k * yb_seg."""
    _abi.call("lx_rowproj_packed_seg", x2.data_ptr(), x2.stride(0), int(x_seg), x2.shape[0], K, wpacks.data_ptr(),
              wpacks[0].numel() if n_seg > 1 else 0, wpacks.shape[3], wpacks.shape[2], r, float(scale), y.data_ptr(),
              y.stride(0), y_seg, _abi.ptr(yb), yb.stride(0) if yb is not None else 0, yb_seg, n_seg,
              _abi.stream_handle(x2.device))


def colgrad_problem(p: torch.Tensor | None, x2: torch.Tensor, ncols: int, r: int, scale: float, out: torch.Tensor,
                    g_sq: int, g_sc: int, masks: NeuronMasks | None = None, blk: int = 1):
    """One G(q, c) = scale * sum_rows P[row, q] X[row, c] problem (c original column) for colgrad_group.
    P may be a column slice (row stride p.stride(0)); X may be a column slice (row stride x2.stride(0))."""
    if p is not None and p.stride(1) != 1:
        p = p.contiguous()
    return dict(p=p, x=x2, ncols=ncols, r=r, scale=float(scale), out=out, g_sq=g_sq, g_sc=g_sc, masks=masks,
                blk=blk if masks is not None else 1)


def colgrad_group(problems: list, n_items: int, s: int) -> None:
    """All problems in one deterministic launch (lx_colgrad_group, up to 16; ranks above 16 split)."""
    flat = []
    for pr in problems:
        r = pr["r"]
        if pr["p"] is not None and r > 16:  # the kernel takes up to 16 ranks per problem
            for q0 in range(0, r, 16):
                sub = dict(pr, p=pr["p"][:, q0:], r=min(16, r - q0))
                sub["out"] = pr["out"].view(-1)[q0 * pr["g_sq"]:] if pr["g_sq"] else pr["out"]
                flat.append(sub)
        else:
            flat.append(pr)
    for i in range(0, len(flat), 16):
        chunk = flat[i : i + 16]
        arr = (_abi.ColgradProblem * len(chunk))()
        keep = []
        for j, pr in enumerate(chunk):
            p, x, m = pr["p"], pr["x"], pr["masks"]
            arr[j] = _abi.ColgradProblem(_abi.ptr(p), p.stride(0) if p is not None else 1, x.data_ptr(), x.stride(0),
                                         pr["ncols"], pr["r"], pr["scale"], _abi.ptr(m.pos if m is not None else None),
                                         pr["blk"], pr["out"].data_ptr(), pr["g_sq"], pr["g_sc"])
            keep.append(p)
        lib = _abi.lib()
        dev = chunk[0]["x"].device
        nws = int(lib.lx_colgrad_group_ws_floats(arr, len(chunk), n_items, s))
        ws = torch.empty(max(nws, 1), dtype=torch.float32, device=dev)
        _abi.call("lx_colgrad_group", arr, len(chunk), n_items, s, ws.data_ptr(), _abi.stream_handle(dev))


def colgrad(p: torch.Tensor | None, x2: torch.Tensor, n_items: int, s: int, ncols: int, r: int, scale: float,
            out: torch.Tensor, g_sq: int, g_sc: int, masks: NeuronMasks | None = None, blk: int = 1) -> torch.Tensor:
    """out(q, c) = scale * sum_rows P[row, q] X[row, c] (c original column), deterministic (one problem)."""
    colgrad_group([colgrad_problem(p, x2, ncols, r, scale, out, g_sq, g_sc, masks, blk)], n_items, s)
    return out
