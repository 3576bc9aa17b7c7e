"""Sequence-oriented runtime sparsity predictors on the B200 (drop-in for the
runtime half of sf/predictor.py:28-168; offline training is out of scope).

Hot path: `attn_pattern_idx` and `mlp_masks` keep everything on the device —
the scoring GEMMs run on tcgen05 and the binarize / OR / upsample / coverage
selection / compaction happen in csrc/mask_build.cu, producing pool indices
and compacted index lists without a host sync. The reference-typed functions
(`predict_attention_patterns` -> list[str], `predict_mlp_mask` -> bool mask)
wrap them and materialise host values only at the API boundary.

Score precision. The reference scores in float32 (sf/predictor.py:74-76,
121-125). The scoring GEMMs carry the fp32 predictor weights as a bf16 hi/lo
pair W = W_hi + W_lo (`k_terms` 2: one K-extended GEMM x [W_hi | W_lo]), which
is exact to ~2^-16 for the bf16 LayerNorm outputs of the fine-tune step; an
fp32 input given to the reference-typed API is split the same way (`k_terms` 3:
[x_hi | x_lo] x [W_hi | W_lo | W_hi]). Masks and patterns then differ from the
float32 reference only where a score lies within that error of its threshold.
`PredictorTrainConfig.score_terms = 1` selects plain bf16 weights (faster,
~2^-9 score error).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _abi
from .neuron_ops import NeuronMasks
from .patterns import DevicePool, LayoutTable, device_pool


def split_bf16(t: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor]:
    """fp32 -> (hi, lo) bf16 with hi + lo = t to ~2^-16 relative."""
    t = t.float()
    hi = t.to(torch.bfloat16)
    return hi, (t - hi.float()).to(torch.bfloat16)


def _pack_terms(w_t: torch.Tensor, terms: int) -> torch.Tensor:
    """fp32 [rows, d] -> bf16 [rows, terms * d]: W (1), [W_hi | W_lo] (2), [W_hi | W_lo | W_hi] (3)."""
    if terms == 1:
        return w_t.to(torch.bfloat16).contiguous()
    hi, lo = split_bf16(w_t)
    return torch.cat([hi, lo] + ([hi] if terms == 3 else []), 1).contiguous()


def _dev_key(device) -> str:
    """Cache key of a device ('cuda' and 'cuda:<current>' are the same device)."""
    dv = torch.device(device)
    if dv.type == "cuda" and dv.index is None:
        dv = torch.device("cuda", torch.cuda.current_device())
    return str(dv)


@dataclass
class AttnPredictorParams:
    """One (wq_hat, wk_hat) low-rank pair per head, each (d, r) (sf/predictor.py:28-37)."""

    wq_hat: list
    wk_hat: list
    _dev: dict = field(default_factory=dict, repr=False)

    @property
    def rank(self) -> int:
        return int(self.wq_hat[0].shape[1])

    def packed_t(self, device, terms: int = 2) -> torch.Tensor:
        """bf16 [2*H*r, terms*d]: rows [h*r, (h+1)*r) = Wq_hat[h]^T, then the Wk_hat[h]^T blocks, as `terms`
        bf16 segments (module docstring). Built once per (device, terms)."""
        key = (_dev_key(device), terms)
        if key not in self._dev:
            def t(w):
                return torch.as_tensor(np.asarray(w) if not torch.is_tensor(w) else w).float().t()
            mats = [t(w) for w in self.wq_hat] + [t(w) for w in self.wk_hat]
            self._dev[key] = _pack_terms(torch.cat(mats, 0).to(device), terms)
        return self._dev[key]


@dataclass
class MlpPredictorParams:
    """wa_hat (d, n_blk) (sf/predictor.py:40-42); device copy is Wa_hat^T bf16 [n_blk, d]."""

    wa_hat: object
    _dev: dict = field(default_factory=dict, repr=False)

    def packed_t(self, device, terms: int = 2) -> torch.Tensor:
        """bf16 [n_blk, terms*d] (module docstring), built once per (device, terms)."""
        key = (_dev_key(device), terms)
        if key not in self._dev:
            w = torch.as_tensor(np.asarray(self.wa_hat) if not torch.is_tensor(self.wa_hat) else self.wa_hat)
            self._dev[key] = _pack_terms(w.float().t().contiguous().to(device), terms)
        return self._dev[key]


@dataclass
class PredictorTrainConfig:
    """Runtime thresholds of sf/predictor.py:45-59 (training fields kept for config compatibility)."""

    noise_std: float = 0.05
    recall_weight: float = 4.0
    epochs: int = 200
    lr: float = 1e-3
    attn_threshold_frac: float = 0.5
    mlp_threshold: float = 0.0
    tau_pred: float = 0.9
    score_terms: int = 2  # device-only: bf16 segments of the predictor weights (module docstring)

    def __post_init__(self):
        if self.noise_std < 0:
            raise ValueError("noise_std must be >= 0")
        if self.recall_weight < 1:
            raise ValueError("recall_weight must be >= 1")


def downsample_indices(s: int) -> np.ndarray:
    """sf/predictor.py:62-67."""
    m = math.isqrt(s)
    if m * m < s:
        m += 1
    return np.minimum((np.arange(m) * s) // m, s - 1)


def downsample(x):
    return x[torch.as_tensor(downsample_indices(x.shape[0]), device=x.device)] if torch.is_tensor(x) else x[downsample_indices(x.shape[0])]


def approx_attention_scores(x_small, wq_hat, wk_hat):
    """sf/predictor.py:74-76 (reference-typed helper, device tensors)."""
    return (x_small @ wq_hat) @ (x_small @ wk_hat).T


def upsample_mask(cell_mask, n_b: int):
    """sf/predictor.py:79-84."""
    m = cell_mask.shape[0]
    src = np.minimum((np.arange(n_b) * m) // n_b, m - 1)
    if torch.is_tensor(cell_mask):
        src = torch.as_tensor(src, device=cell_mask.device)
        return cell_mask[src][:, src]
    return cell_mask[np.ix_(src, src)]


def binarize_scores(s_hat, threshold_frac: float):
    """sf/predictor.py:87-90 (threshold rounded in the score dtype, strict '>')."""
    if torch.is_tensor(s_hat):
        peak = s_hat.max()
        return s_hat > (torch.tensor(threshold_frac, dtype=s_hat.dtype, device=s_hat.device) * peak)
    return s_hat > (s_hat.dtype.type(threshold_frac) * s_hat.max())


# ---------------------------------------------------------------- device hot path


def _pool_dev(pool, device) -> DevicePool:
    if isinstance(pool, DevicePool):
        return pool
    cache = _pool_dev.__dict__.setdefault("cache", {})
    key = (id(pool), str(device))
    if key not in cache:
        cache[key] = (pool, device_pool(pool, device))
    return cache[key][1]


def _terms_input(x: torch.Tensor, terms: int) -> tuple[torch.Tensor, int, int]:
    """Scoring-GEMM input for `terms`: bf16 x (terms 1, 2; an fp32 x is rounded), or [x_hi | x_lo] for 3.
    Split terms need d % 64 == 0: a narrower d falls back to one term. Returns (input, d, terms)."""
    d = x.shape[1]
    if terms > 1 and d % 64:
        terms = 1
    if terms == 3:
        hi, lo = split_bf16(x)
        return torch.cat([hi, lo], 1).contiguous(), d, 3
    return x.to(torch.bfloat16).contiguous(), d, terms


def attn_pattern_idx(x_small: torch.Tensor, n_items: int, m: int, params: AttnPredictorParams, pool, n_b: int,
                     cfg: PredictorTrainConfig, scope_batch: bool = False, dump: bool = False, terms: int | None = None):
    """Fused K1a: x_small [n_items*m, d] (bf16; fp32 with terms=3) -> pool index int32 [n_items (or 1), H] on
    device. Returns (idx, scores [n_items, H, m, m] fp32 or None)."""
    dev = x_small.device
    dp = _pool_dev(pool, dev)
    x_small, d, terms = _terms_input(x_small, cfg.score_terms if terms is None else terms)
    H, r = len(params.wq_hat), params.rank
    wqk = params.packed_t(dev, terms)
    proj = torch.empty(n_items * m, 2 * H * r, dtype=torch.float32, device=dev)
    idx = torch.empty(1 if scope_batch else n_items, H, dtype=torch.int32, device=dev)
    sc = torch.empty(n_items, H, m, m, dtype=torch.float32, device=dev) if dump else None
    _abi.call("lx_predict_attention_patterns", x_small.data_ptr(), n_items, m, d, wqk.data_ptr(), H, r, terms,
              float(np.float32(cfg.attn_threshold_frac)), float(cfg.tau_pred), n_b, dp.kinds.data_ptr(),
              dp.params.data_ptr(), len(dp.ids), int(scope_batch), proj.data_ptr(), idx.data_ptr(), _abi.ptr(sc),
              _abi.stream_handle(dev))
    return idx, sc


def mlp_masks(h: torch.Tensor, n_items: int, s: int, params: MlpPredictorParams, threshold: float, blk: int,
              scope_batch: bool = False, dump: bool = False, terms: int = 2):
    """Fused K1b: h [n_items*s, d] (bf16; fp32 with terms=3) -> NeuronMasks (counts/ids/pos) on device.
    Returns (masks, scores fp32 [n_items*s, n_blk] or None)."""
    dev = h.device
    h, d, terms = _terms_input(h, terms)
    wa = params.packed_t(dev, terms)
    n_blk = wa.shape[0]
    words = (n_blk + 31) // 32
    bits = torch.empty(n_items, (s + 31) // 32, words, dtype=torch.int32, device=dev)  # per 32-row slot, all stored
    counts = torch.empty(n_items, dtype=torch.int32, device=dev)
    ids = torch.empty(n_items, n_blk, dtype=torch.int32, device=dev)  # tail zeroed by the compaction kernel
    pos = torch.empty(n_items, n_blk, dtype=torch.int32, device=dev)
    sc = torch.empty(n_items * s, n_blk, dtype=torch.float32, device=dev) if dump else None
    _abi.call("lx_predict_mlp_mask", h.data_ptr(), n_items, s, d, wa.data_ptr(), n_blk, terms, float(threshold), int(scope_batch),
              bits.data_ptr(), counts.data_ptr(), ids.data_ptr(), pos.data_ptr(), _abi.ptr(sc), _abi.stream_handle(dev))
    return NeuronMasks(counts, ids, pos, n_blk, blk), sc


def x_small_of(x_batch: torch.Tensor, keep_dtype: bool = False) -> tuple[torch.Tensor, int]:
    """Downsampled rows of every item (sf/predictor.py:62-71): [B, s, d] -> ([B*m, d] bf16 (or the input
    dtype with keep_dtype), m)."""
    B, s, d = x_batch.shape
    idx = torch.as_tensor(downsample_indices(s), device=x_batch.device)
    xs = x_batch[:, idx, :]
    if not keep_dtype:
        xs = xs.to(torch.bfloat16)
    return xs.reshape(B * len(idx), d).contiguous(), len(idx)


def _stack(x_batch) -> torch.Tensor:
    if torch.is_tensor(x_batch):
        return x_batch if x_batch.dim() == 3 else x_batch[None]
    return torch.stack([torch.as_tensor(np.asarray(x)) if not torch.is_tensor(x) else x for x in x_batch])


def predict_attention_patterns(x_batch, params: AttnPredictorParams, pool: dict[str, LayoutTable],
                               cfg: PredictorTrainConfig, counter=None) -> list[str]:
    """sf/predictor.py:93-118: per-head pattern ids for a batch (OR over the batch). Float32 inputs are scored at
    float32 precision (k_terms 3), bf16 inputs with the split weights (k_terms 2)."""
    xb = _stack(x_batch)
    dev = xb.device if xb.is_cuda else torch.device("cuda")
    xs, m = x_small_of(xb.to(dev), keep_dtype=True)
    n_b = next(iter(pool.values())).n_b
    terms = 3 if xs.dtype == torch.float32 and cfg.score_terms > 1 else cfg.score_terms
    idx, _ = attn_pattern_idx(xs, xb.shape[0], m, params, pool, n_b, cfg, scope_batch=True, terms=terms)
    if counter is not None:
        d, r = xb.shape[2], params.rank
        counter.add(xb.shape[0] * len(params.wq_hat) * (2 * m * d * r + m * m * r))
    ids = list(pool)
    return [ids[i] for i in idx[0].tolist()]


def approx_mlp_scores(x, params: MlpPredictorParams, counter=None, terms: int = 3) -> torch.Tensor:
    """sf/predictor.py:121-125: S_hat = X Wa_hat (fp32 out of the tcgen05 GEMM; a float32 X and the fp32 weights
    as bf16 hi/lo pairs, k_terms 3: float32-level scores)."""
    xt = torch.as_tensor(np.asarray(x)) if not torch.is_tensor(x) else x
    xt = xt.to("cuda" if not xt.is_cuda else xt.device)
    if xt.dtype == torch.bfloat16:
        terms = min(terms, 2)
    xi, d, terms = _terms_input(xt.float() if terms == 3 else xt, terms)
    wa = params.packed_t(xt.device, terms)
    n_blk = wa.shape[0]
    out = torch.empty(xt.shape[0], n_blk, dtype=torch.float32, device=xt.device)
    _abi.call("lx_gemm_bf16_tn", xi.data_ptr(), xi.shape[1], wa.data_ptr(), wa.shape[1], out.data_ptr(), n_blk, 1,
              xt.shape[0], n_blk, terms * d, d if terms > 1 else 0, _abi.stream_handle(xt.device))
    if counter is not None:
        counter.add(xt.shape[0] * d * n_blk)
    return out


def predict_mlp_mask(s_hat_batch, threshold: float, counter=None) -> torch.Tensor:
    """sf/predictor.py:128-139: (S > thr).any(axis=0), OR over items (reference-typed)."""
    mask = None
    for s_hat in s_hat_batch:
        st = s_hat if torch.is_tensor(s_hat) else torch.as_tensor(np.asarray(s_hat))
        a = (st > threshold).any(dim=0)
        if counter is not None:
            counter.add(st.shape[0])
        mask = a if mask is None else (mask | a)
    if mask is None:
        raise ValueError("empty batch")
    return mask


def eval_recall_precision(predicted, truth) -> tuple[float, float]:
    """sf/predictor.py:142-150."""
    p = np.asarray(predicted.cpu() if torch.is_tensor(predicted) else predicted, dtype=bool)
    t = np.asarray(truth.cpu() if torch.is_tensor(truth) else truth, dtype=bool)
    if p.shape != t.shape:
        raise ValueError("mask lengths differ")
    hit = (p & t).sum()
    return (float(hit / t.sum()) if t.any() else 1.0, float(hit / p.sum()) if p.any() else 1.0)


def predictor_cost_flops(s: int, d: int, r: int) -> tuple[int, int]:
    """sf/predictor.py:153-168 (analytic MACs)."""
    if s < 1 or d < 1 or r < 1:
        raise ValueError("sizes must be positive")
    root = math.isqrt(s)
    if root * root < s:
        root += 1
    return root * d * r * 2 + s * r, s * d * r + s
