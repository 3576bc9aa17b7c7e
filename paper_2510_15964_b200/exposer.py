"""Exposer oracle mode on the GPU (sf/exposer.py:33-171; its providers sf/harness.py:157-190).

The dense ground truth the predicted masks approximate: exact per-head attention
probabilities summed into block masses, the fewest-block pool pattern covering tau
of the mass, and peak-relative neuron-block filtering of the exact MLP
pre-activation. Verification mode — it pays the dense cost the hot path avoids —
so the projections are plain cuBLAS GEMMs and the sparsity-specific work runs in
csrc/exposer.cu: `lx_exact_block_mass` (fp32 dot products, float64 softmax and
block sums like the reference), `lx_select_by_coverage` (bit-identical choice for
a given grid), `lx_block_importance` + `lx_filter_neuron_blocks` (+ the shared
`lx_mask_compact`). Results stay on the device in the same forms the predicted
provider returns (pool indices [B, H], NeuronMasks), so the fine-tune step and
its CUDA graph take either.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _abi, model as M
from .errors import PatternError, ShapeError
from .neuron_ops import NeuronMasks


def shadowy_combine(per_token_active) -> np.ndarray:
    """sf/exposer.py:19-30 (host helper: OR of per-token activity vectors)."""
    if not len(per_token_active):
        raise ValueError("need at least one per-token activity vector")
    out = np.asarray(per_token_active[0], dtype=bool).copy()
    for vec in per_token_active[1:]:
        vec = np.asarray(vec, dtype=bool)
        if vec.shape != out.shape:
            raise ValueError("activity vectors differ in length")
        out |= vec
    return out


def sparsity_ratio(mask) -> float:
    """sf/exposer.py:33-38."""
    mask = mask.cpu().numpy() if torch.is_tensor(mask) else np.asarray(mask)
    mask = mask.astype(bool)
    if mask.size == 0:
        raise ValueError("empty mask")
    return float(1.0 - mask.sum() / mask.size)


def exact_qk(h: torch.Tensor, lw: M.LayerWeights) -> torch.Tensor:
    """[q | k] = h [W_Q | W_K] + [b_Q | b_K] (frozen weights, no LoRA: sf/exposer.py:49-50), fp32 [M, 2d]."""
    d = lw.d
    h2 = h.reshape(-1, h.shape[-1]).to(torch.bfloat16)
    return M._mm_f32(h2, lw.wqkv[:, : 2 * d]).add_(lw.bqkv[: 2 * d])


def exact_block_mass(qk: torch.Tensor, n_items: int, s: int, n_heads: int, n_b: int) -> torch.Tensor:
    """exact_attention + block_mass (sf/exposer.py:47-68) from fp32 projections [n_items*s, 2d]
    (q columns [0, d), k columns [d, 2d)): float64 [n_items, H, n_b, n_b]."""
    if qk.dtype != torch.float32 or qk.dim() != 2 or qk.shape[0] != n_items * s or qk.shape[1] % 2:
        raise ShapeError(f"qk must be fp32 [n_items*s, 2d], got {tuple(qk.shape)} {qk.dtype}")
    qk = qk.contiguous()
    d = qk.shape[1] // 2
    if d % n_heads:
        raise ShapeError(f"d={d} not divisible by {n_heads} heads")
    mass = torch.empty(n_items, n_heads, n_b, n_b, dtype=torch.float64, device=qk.device)
    _abi.call("lx_exact_block_mass", qk.data_ptr(), qk.data_ptr() + 4 * d, 2 * d, n_items, s, n_heads, d // n_heads, n_b,
              mass.data_ptr(), _abi.stream_handle(qk.device))
    return mass


def select_by_coverage(mass: torch.Tensor, dpool, tau: float, head_sum: bool = False) -> torch.Tensor:
    """select_pattern_by_coverage per (item, head) grid (sf/exposer.py:71-91), or once per item over
    the head-summed grids (ShadowyProvider, sf/harness.py:183-187): int32 pool indices [B, H]."""
    if not (0 < tau <= 1):
        raise ValueError(f"coverage tau must be in (0, 1], got {tau}")
    if dpool.ids[-1] != "dense":
        raise PatternError("the device coverage selection falls back to the pool's last entry, which must be 'dense'")
    B, H, n_b, _ = mass.shape
    mass = mass.to(torch.float64).contiguous()
    idx = torch.empty(B, H, dtype=torch.int32, device=mass.device)
    _abi.call("lx_select_by_coverage", mass.data_ptr(), B, H, n_b, dpool.kinds.data_ptr(), dpool.params.data_ptr(),
              len(dpool.ids), float(tau), int(head_sum), idx.data_ptr(), _abi.stream_handle(mass.device))
    return idx


def mlp_preactivation(h: torch.Tensor, lw: M.LayerWeights, adapter=None) -> torch.Tensor:
    """z = h W1 + b1 (+ scaling (h A) B) (sf/harness.py:170-174), fp32 [M, d_ff]."""
    h2 = h.reshape(-1, h.shape[-1]).to(torch.bfloat16)
    z = M._mm_f32(h2, lw.mlp.w1).add_(lw.b1)
    if adapter is not None:
        z.add_((h2.float() @ adapter.a) @ adapter.b, alpha=float(adapter.scaling))
    return z


def block_importance(z: torch.Tensor, n_items: int, s: int, blk: int) -> torch.Tensor:
    """sf/exposer.py:94-98 per item: fp32 [n_items, ceil(n_cols / blk)], max |relu(z)| per block."""
    if z.dtype != torch.float32 or z.dim() != 2 or z.shape[0] != n_items * s:
        raise ShapeError(f"z must be fp32 [n_items*s, n_cols], got {tuple(z.shape)} {z.dtype}")
    if z.stride(1) != 1:
        z = z.contiguous()
    n_cols = z.shape[1]
    imp = torch.empty(n_items, -(-n_cols // blk), dtype=torch.float32, device=z.device)
    _abi.call("lx_block_importance", z.data_ptr(), z.stride(0), n_items, s, n_cols, blk, imp.data_ptr(),
              _abi.stream_handle(z.device))
    return imp


def filter_neuron_blocks(imp: torch.Tensor, theta: float, blk: int) -> NeuronMasks:
    """sf/exposer.py:101-111 per item, lowered to NeuronMasks (ascending ids, counts, positions)."""
    if not (0 <= theta <= 1):
        raise ValueError(f"theta must be in [0, 1], got {theta}")
    B, n_blk = imp.shape
    dev = imp.device
    bits = torch.empty(B, (n_blk + 31) // 32, dtype=torch.int32, device=dev)
    counts = torch.empty(B, dtype=torch.int32, device=dev)
    ids = torch.empty(B, n_blk, dtype=torch.int32, device=dev)
    pos = torch.empty(B, n_blk, dtype=torch.int32, device=dev)
    st = _abi.stream_handle(dev)
    _abi.call("lx_filter_neuron_blocks", imp.contiguous().data_ptr(), B, n_blk, float(theta), bits.data_ptr(), st)
    _abi.call("lx_mask_compact", bits.data_ptr(), B, n_blk, 0, counts.data_ptr(), ids.data_ptr(), pos.data_ptr(), st)
    return NeuronMasks(counts, ids, pos, n_blk, blk)


def head_masks_and_union(idx_row, pool) -> tuple[list[str], np.ndarray]:
    """sf/exposer.py:114-123 for one item's pool indices."""
    ids = list(pool)
    assignment = [ids[int(i)] for i in idx_row]
    n_b = next(iter(pool.values())).n_b
    union = np.zeros((n_b, n_b), dtype=bool)
    for pid in assignment:
        for br, bc in pool[pid].coords:
            union[br, bc] = True
    return assignment, union


class _Recorder:
    """Dense masks that keep each layer's attention / MLP inputs (the exposer's layer_activations,
    sf/exposer.py:126-140, without a second forward)."""

    fused_downsample = False

    def __init__(self, model: M.Model):
        self.model, self.h_attn, self.h_mlp = model, {}, {}

    def attn_patterns(self, layer, h, x_small=None):
        self.h_attn[layer] = h
        return ["dense"] * self.model.dims.n_heads

    def mlp_mask(self, layer, h):
        self.h_mlp[layer] = h
        return np.ones(self.model.dims.n_blk, dtype=bool)


@torch.no_grad()
def layer_sparsity_report(model: M.Model, tokens, thetas, tau: float = 0.95) -> list[dict]:
    """sf/exposer.py:143-164: per-layer shadowy / head-specific attention sparsity and shadowy /
    theta-filtered MLP sparsity of one sequence (tokens [s]), CSV-ready rows."""
    tok = torch.as_tensor(np.asarray(tokens), dtype=torch.int64, device=model.device).reshape(1, -1)
    rec = _Recorder(model)
    M.model_forward(model, tok, rec)
    dims, s = model.dims, tok.shape[1]
    rows = []
    for layer in range(dims.n_layers):
        lw = model.weights.layers[layer]
        mass = exact_block_mass(exact_qk(rec.h_attn[layer], lw), 1, s, dims.n_heads, dims.n_b)
        idx = select_by_coverage(mass, model.dpool, tau)
        assignment, union = head_masks_and_union(idx[0].tolist(), model.pool)
        head_active = sum(model.pool[pid].active_blocks for pid in assignment)
        rows.append({"layer": layer, "component": "attention", "method": "shadowy", "theta": 0.0,
                     "sparsity_ratio": sparsity_ratio(np.tile(union, (dims.n_heads, 1)))})
        rows.append({"layer": layer, "component": "attention", "method": "head_specific", "theta": 0.0,
                     "sparsity_ratio": 1.0 - head_active / (dims.n_heads * dims.n_b**2)})
        ad = model.lora.get((layer, "w1")) if model.peft_method == "lora" else None
        z = mlp_preactivation(rec.h_mlp[layer], lw, ad)
        # neuron-level shadowy activity: a neuron is active iff some token has z > 0 (blk = 1 importance)
        seq_active = block_importance(z, 1, s, 1)[0] > 0
        rows.append({"layer": layer, "component": "mlp", "method": "shadowy", "theta": 0.0,
                     "sparsity_ratio": sparsity_ratio(seq_active)})
        imp = block_importance(z, 1, s, dims.blk_size)
        for theta in thetas:
            nm = filter_neuron_blocks(imp, float(theta), dims.blk_size)
            rows.append({"layer": layer, "component": "mlp", "method": "neuron_filter", "theta": float(theta),
                         "sparsity_ratio": sparsity_ratio(nm.to_bool())})
    return rows


def report_to_csv(rows: list[dict]) -> str:
    """sf/exposer.py:167-171."""
    lines = ["layer,component,method,theta,sparsity_ratio"]
    for r in rows:
        lines.append(f"{r['layer']},{r['component']},{r['method']},{r['theta']:.6f},{r['sparsity_ratio']:.6f}")
    return "\n".join(lines) + "\n"
