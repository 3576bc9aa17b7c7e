"""TEST INFRASTRUCTURE ONLY — NumPy restatement of the reference hot path.

Every function restates the algorithm of the reference module cited in its
docstring (``sf/`` = /root/reference/pkg/src/sparseft/). The block-sparse
operators are vectorised over blocks (gather -> batched matmul -> segmented
reduce) instead of the reference's per-block Python loop; the arithmetic per
block (what is multiplied with what, where the max-shift and the -inf mask
apply, which entries receive gradient) is identical, so results agree to
float rounding. Integer / boolean mask logic is restated exactly, including
NumPy-2 scalar promotion (NEP 50) in ``binarize_scores`` and the sequential
float64 coverage sum in ``select_pattern_by_coverage``.

Not shipped; see oracle/__init__.py for who may import this.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np


# ---------------------------------------------------------------------------
# error types (same names / ValueError bases as the reference)


class PatternError(ValueError):
    """sf/patterns.py:20"""


class LayoutError(ValueError):
    """sf/block_sparse.py:18"""


class MaskError(ValueError):
    """sf/neuron_ops.py:18"""


class ShapeError(ValueError):
    """sf/tensor_core.py:15"""


class GradientError(ValueError):
    """sf/autograd.py:24"""


def make_rng(seed: int) -> np.random.Generator:
    """sf/tensor_core.py:19-21 — seeded PCG64."""
    return np.random.Generator(np.random.PCG64(seed))


def randn(rng, shape, scale: float) -> np.ndarray:
    """sf/tensor_core.py:24-28."""
    if scale <= 0:
        raise ValueError("scale must be > 0")
    return (rng.standard_normal(shape) * scale).astype(np.float32)


# ---------------------------------------------------------------------------
# pattern pool (sf/patterns.py:63-133)


def _pattern_cells(kind: str, n_b: int, p: int = 0) -> np.ndarray:
    """Boolean n_b x n_b grid of one atomic pattern (sf/patterns.py:63-85)."""
    i = np.arange(n_b)[:, None]
    j = np.arange(n_b)[None, :]
    if kind == "blockdiag":
        g = i == j
    elif kind == "band":
        g = np.abs(i - j) <= p
    elif kind == "causal":
        g = (i - j >= 0) & (i - j <= p)
    elif kind == "global":
        g = (i < p) | (j < p) | (i == j)
    elif kind == "strided":
        g = (i - j) % p == 0
    elif kind == "dense":
        g = np.ones((n_b, n_b), dtype=bool)
    else:  # pragma: no cover
        raise PatternError(kind)
    return np.broadcast_to(g, (n_b, n_b))


def build_pool(n_b: int, band_widths=(1, 2), global_sizes=(1,), strides=(2,), causal_widths=(1,)) -> dict:
    """sf/patterns.py:88-120. Returns ordered {pattern_id: int32 coords [nnz, 2]}
    with coordinates sorted row-major (the reference's sorted tuple order)."""
    if n_b < 1:
        raise PatternError(f"grid side must be >= 1, got {n_b}")
    specs = [("blockdiag", "blockdiag", 0)]
    for w in band_widths:
        if w > n_b:
            raise PatternError(f"band width {w} exceeds grid side {n_b}")
        specs.append((f"band{w}", "band", w))
    for w in causal_widths:
        if w > n_b:
            raise PatternError(f"causal width {w} exceeds grid side {n_b}")
        specs.append((f"causal{w}", "causal", w))
    for g in global_sizes:
        if g > n_b:
            raise PatternError(f"global border {g} exceeds grid side {n_b}")
        specs.append((f"global{g}", "global", g))
    for p in strides:
        if p > n_b:
            raise PatternError(f"stride {p} exceeds grid side {n_b}")
        specs.append((f"strided{p}", "strided", p))
    specs.append(("dense", "dense", 0))
    pool: dict[str, np.ndarray] = {}
    for pid, kind, p in specs:
        if pid in pool:
            continue
        br, bc = np.nonzero(_pattern_cells(kind, n_b, p))  # row-major == sorted order
        pool[pid] = np.stack([br, bc], axis=1).astype(np.int32)
    return pool


def combine_layouts(assignment, pool) -> tuple[np.ndarray, np.ndarray]:
    """sf/patterns.py:123-133. Returns (entries [E,3] (head, br, bc), head_offsets [H])."""
    entries, offsets, n = [], [], 0
    for h, pid in enumerate(assignment):
        if pid not in pool:
            raise PatternError(f"pattern id {pid!r} not in pool")
        c = pool[pid]
        offsets.append(n)
        entries.append(np.concatenate([np.full((len(c), 1), h, np.int32), c], axis=1))
        n += len(c)
    ent = np.concatenate(entries) if entries else np.zeros((0, 3), np.int32)
    return ent, np.asarray(offsets, dtype=np.int64)


# ---------------------------------------------------------------------------
# predictor runtime (sf/predictor.py:62-139) and exposer selection (sf/exposer.py)


def downsample_indices(s: int) -> np.ndarray:
    """sf/predictor.py:62-67: m = ceil(sqrt(s)) rows at min(i*s//m, s-1)."""
    m = math.isqrt(s)
    m += int(m * m < s)
    return np.minimum((np.arange(m) * s) // m, s - 1)


def approx_attention_scores(x_small, wq_hat, wk_hat):
    """sf/predictor.py:74-76."""
    return (x_small @ wq_hat) @ (x_small @ wk_hat).T


def upsample_mask(cell_mask: np.ndarray, n_b: int) -> np.ndarray:
    """sf/predictor.py:79-84: nearest cell min(i*m//n_b, m-1) (subsamples when m > n_b)."""
    m = cell_mask.shape[0]
    src = np.minimum((np.arange(n_b) * m) // n_b, m - 1)
    return cell_mask[src][:, src]


def binarize_scores(s_hat: np.ndarray, threshold_frac: float) -> np.ndarray:
    """sf/predictor.py:87-90. NEP 50: the Python-float fraction is cast to the
    score dtype before the multiply, so the threshold is rounded in fp32 for
    fp32 scores; strict '>'."""
    peak = s_hat.max()
    thr = s_hat.dtype.type(threshold_frac) * peak
    return s_hat > thr


def select_pattern_by_coverage(grid_weight: np.ndarray, pool: dict, tau: float) -> str:
    """sf/exposer.py:71-85. Fewest-blocks pattern with mass/total >= tau - 1e-9
    (float64), ties by pool order; zero total or no candidate -> 'dense'."""
    if not (0 < tau <= 1):
        raise ValueError(f"coverage tau must be in (0, 1], got {tau}")
    total = grid_weight.sum()
    if total <= 0:
        return "dense"
    best, best_n = None, None
    for pid, coords in pool.items():
        vals = grid_weight[coords[:, 0], coords[:, 1]]
        mass = np.cumsum(vals)[-1] if len(vals) else 0.0  # sequential left-to-right sum
        if mass / total >= tau - 1e-9 and (best is None or len(coords) < best_n):
            best, best_n = pid, len(coords)
    return best if best is not None else "dense"


@dataclass
class AttnPredictorParams:
    """sf/predictor.py:28-37 — per head (d, r) factors."""

    wq_hat: list
    wk_hat: list


@dataclass
class MlpPredictorParams:
    """sf/predictor.py:40-42 — (d, n_blk)."""

    wa_hat: np.ndarray


@dataclass
class PredictorConfig:
    """Runtime thresholds of sf/predictor.py:45-59."""

    attn_threshold_frac: float = 0.5
    mlp_threshold: float = 0.0
    tau_pred: float = 0.9


def predict_attention_patterns(x_batch, params: AttnPredictorParams, pool, cfg: PredictorConfig, return_scores=False):
    """sf/predictor.py:93-118: binarize per item, OR over batch, upsample, categorize."""
    n_b = int(np.sqrt(len(pool["dense"])))
    out, scores = [], []
    for h in range(len(params.wq_hat)):
        active = None
        for x in x_batch:
            xs = x[downsample_indices(x.shape[0])]
            s_hat = approx_attention_scores(xs, params.wq_hat[h], params.wk_hat[h])
            scores.append(s_hat)
            cell = binarize_scores(s_hat, cfg.attn_threshold_frac)
            active = cell if active is None else (active | cell)
        grid = upsample_mask(active, n_b).astype(np.float64)
        out.append(select_pattern_by_coverage(grid, pool, cfg.tau_pred))
    return (out, scores) if return_scores else out


def patterns_from_scores(score_maps, n_b: int, pool, cfg: PredictorConfig) -> list[str]:
    """The mask-build tail of sf/predictor.py:114-117 applied to given score maps
    (one [m, m] map per head, single item): the bit-exactness check point."""
    return [
        select_pattern_by_coverage(upsample_mask(binarize_scores(s, cfg.attn_threshold_frac), n_b).astype(np.float64), pool, cfg.tau_pred)
        for s in score_maps
    ]


def approx_mlp_scores(x, params: MlpPredictorParams):
    """sf/predictor.py:121-125."""
    return x @ params.wa_hat


def predict_mlp_mask(s_hat_batch, threshold: float) -> np.ndarray:
    """sf/predictor.py:128-139: (S > thr).any(axis=0), OR over items."""
    mask = None
    for s in s_hat_batch:
        a = (s > threshold).any(axis=0)
        mask = a if mask is None else (mask | a)
    if mask is None:
        raise ValueError("empty batch")
    return mask


def shadowy_combine(per_token_active) -> np.ndarray:
    """sf/exposer.py:19-30."""
    if len(per_token_active) == 0:
        raise ValueError("need at least one per-token activity vector")
    arr = [np.asarray(v, dtype=bool) for v in per_token_active]
    if any(a.shape != arr[0].shape for a in arr):
        raise ValueError("activity vectors differ in length")
    return np.logical_or.reduce(np.stack(arr), axis=0)


def sparsity_ratio(mask) -> float:
    """sf/exposer.py:33-38."""
    mask = np.asarray(mask, dtype=bool)
    if mask.size == 0:
        raise ValueError("empty mask")
    return float(1.0 - mask.sum() / mask.size)


def block_importance(z: np.ndarray, blk_size: int) -> np.ndarray:
    """sf/exposer.py:94-98: max |relu(z)| per neuron block (ragged tail allowed)."""
    act = np.maximum(z, 0)
    n_blk = -(-z.shape[1] // blk_size)
    return np.array([act[:, b * blk_size : (b + 1) * blk_size].max() if act.shape[0] else 0.0 for b in range(n_blk)])


def filter_neuron_blocks(importance, theta: float) -> np.ndarray:
    """sf/exposer.py:101-111 (float64 compare against theta * peak)."""
    if not (0 <= theta <= 1):
        raise ValueError(f"theta must be in [0, 1], got {theta}")
    imp = np.asarray(importance, dtype=np.float64)
    peak = imp.max() if imp.size else 0.0
    if peak <= 0:
        return np.zeros(imp.shape, dtype=bool)
    return imp > theta * peak


def block_mass(weight: np.ndarray, n_b: int) -> np.ndarray:
    """sf/exposer.py:62-68."""
    s = weight.shape[0]
    blk = s // n_b
    if blk * n_b != s:
        raise ValueError(f"matrix side {s} not divisible by grid side {n_b}")
    return weight.reshape(n_b, blk, n_b, blk).sum(axis=(1, 3))


def exact_attention(x, wq, bq, wk, bk, n_heads: int):
    """sf/exposer.py:47-59: per-head (probabilities, raw scores). q, k in the input dtype; the
    np.float64 scale 1/sqrt(head_dim) promotes raw scores (and so the softmax) to float64."""
    q = x @ wq + bq
    k = x @ wk + bk
    return exact_attention_qk(q, k, n_heads)


def exact_attention_qk(q, k, n_heads: int):
    """exact_attention from given projections (sf/exposer.py:51-59; softmax sf/tensor_core.py:85-91)."""
    hd = q.shape[1] // n_heads
    scale = 1.0 / np.sqrt(hd)
    probs, raws = [], []
    for h in range(n_heads):
        sl = slice(h * hd, (h + 1) * hd)
        raw = (q[:, sl] @ k[:, sl].T) * scale
        sh = raw - raw.max(axis=1, keepdims=True)
        e = np.exp(sh)
        raws.append(raw)
        probs.append(e / e.sum(axis=1, keepdims=True))
    return probs, raws


def select_head_pattern(probs_h, pool: dict, tau: float = 0.95) -> str:
    """sf/exposer.py:88-91."""
    n_b = _pool_nb(pool)
    return select_pattern_by_coverage(block_mass(probs_h, n_b), pool, tau)


def _pool_nb(pool: dict) -> int:
    """Grid side of a pool (its dense pattern holds every cell)."""
    return int(round(math.sqrt(len(pool["dense"]))))


def shadowy_pattern(probs, pool: dict, tau: float) -> str:
    """ShadowyProvider._attn (sf/harness.py:183-187): one pattern for all heads from the summed masses."""
    n_b = _pool_nb(pool)
    mass = sum(block_mass(p, n_b) for p in probs)
    return select_pattern_by_coverage(mass, pool, tau)


def oracle_mlp_mask(h, w1, b1, lora_a, lora_b, scaling, blk: int, theta: float):
    """OracleProvider._mlp (sf/harness.py:169-176): z = h W1 + b1 (+ s (h A) B), importance, filter."""
    z = h @ w1 + b1
    if lora_a is not None:
        z = z + scaling * ((h @ lora_a) @ lora_b)
    return filter_neuron_blocks(block_importance(z, blk), theta), z


# ---------------------------------------------------------------------------
# block-sparse attention operators (sf/block_sparse.py:47-150), vectorised


def _check_grid(s, blk, coords, n_b):
    """sf/block_sparse.py:39-44."""
    if s != n_b * blk:
        raise LayoutError(f"sequence length {s} != n_b*blk = {n_b}*{blk}")
    c = np.asarray(coords).reshape(-1, 2)
    if c.size and (c.min() < 0 or c.max() >= n_b):
        raise LayoutError("block outside grid")
    return c


def sdd(q, k, coords, blk, scale):
    """sf/block_sparse.py:47-60: scale * Q_br K_bc^T for each active block, layout order."""
    s, hd = q.shape
    n_b = s // blk
    c = _check_grid(s, blk, coords, n_b)
    qb = q.reshape(n_b, blk, hd)[c[:, 0]]
    kb = k.reshape(n_b, blk, hd)[c[:, 1]]
    return (qb @ kb.transpose(0, 2, 1)) * scale


def sparse_softmax(blocks, coords, n_b):
    """sf/block_sparse.py:81-99: per token row, softmax over the union of the
    block-row's active blocks; an uncovered block-row raises LayoutError."""
    c = np.asarray(coords).reshape(-1, 2)
    br = c[:, 0]
    covered = np.zeros(n_b, dtype=bool)
    covered[br] = True
    if not covered.all():
        raise LayoutError(f"block-row {int(np.flatnonzero(~covered)[0])} has no active blocks (pattern pool violation)")
    blk = blocks.shape[1]
    rmax = np.full((n_b, blk), -np.inf, dtype=blocks.dtype)
    np.maximum.at(rmax, br, blocks.max(axis=2))
    e = np.exp(blocks - rmax[br][:, :, None])
    den = np.zeros((n_b, blk), dtype=blocks.dtype)
    np.add.at(den, br, e.sum(axis=2))
    return e / den[br][:, :, None]


def sparse_softmax_backward(p_blocks, d_blocks, coords, n_b):
    """sf/block_sparse.py:102-113: ds = p * (dp - rowsum(dp*p))."""
    br = np.asarray(coords).reshape(-1, 2)[:, 0]
    inner = np.zeros((n_b, p_blocks.shape[1]), dtype=p_blocks.dtype)
    np.add.at(inner, br, (d_blocks * p_blocks).sum(axis=2))
    return p_blocks * (d_blocks - inner[br][:, :, None])


def dsd(p_blocks, v, coords, n_b):
    """sf/block_sparse.py:116-126: out[br] += P_blk V_bc."""
    s, hd = v.shape
    blk = p_blocks.shape[1]
    if s != n_b * blk:
        raise LayoutError(f"value rows {s} != grid {n_b}*{blk}")
    c = np.asarray(coords).reshape(-1, 2)
    prod = p_blocks @ v.reshape(n_b, blk, hd)[c[:, 1]]
    out = np.zeros((n_b, blk, hd), dtype=np.result_type(p_blocks, v))
    np.add.at(out, c[:, 0], prod)
    return out.reshape(s, hd)


def dsd_backward(p_blocks, v, d_out, coords, n_b):
    """sf/block_sparse.py:129-137: dP_blk = dO_br V_bc^T; dV_bc += P_blk^T dO_br."""
    s, hd = v.shape
    blk = p_blocks.shape[1]
    c = np.asarray(coords).reshape(-1, 2)
    g = d_out.reshape(n_b, blk, hd)[c[:, 0]]
    d_blocks = g @ v.reshape(n_b, blk, hd)[c[:, 1]].transpose(0, 2, 1)
    dv = np.zeros((n_b, blk, hd), dtype=v.dtype)
    np.add.at(dv, c[:, 1], p_blocks.transpose(0, 2, 1) @ g)
    return d_blocks, dv.reshape(s, hd)


def sdd_backward(d_blocks, q, k, coords, blk, scale):
    """sf/block_sparse.py:63-71: dQ_br += scale dS K_bc; dK_bc += scale dS^T Q_br."""
    s, hd = q.shape
    n_b = s // blk
    c = np.asarray(coords).reshape(-1, 2)
    g = d_blocks * scale
    dq = np.zeros((n_b, blk, hd), dtype=q.dtype)
    dk = np.zeros((n_b, blk, hd), dtype=k.dtype)
    np.add.at(dq, c[:, 0], g @ k.reshape(n_b, blk, hd)[c[:, 1]])
    np.add.at(dk, c[:, 1], g.transpose(0, 2, 1) @ q.reshape(n_b, blk, hd)[c[:, 0]])
    return dq.reshape(s, hd), dk.reshape(s, hd)


def dense_masked_attention(q, k, v, coords, blk, scale):
    """sf/block_sparse.py:140-150: float64 -inf-masked dense oracle."""
    s = q.shape[0]
    mask = np.full((s, s), -np.inf)
    for br, bc in np.asarray(coords).reshape(-1, 2):
        mask[br * blk : (br + 1) * blk, bc * blk : (bc + 1) * blk] = 0.0
    sc = (q.astype(np.float64) @ k.astype(np.float64).T) * scale + mask
    e = np.where(np.isfinite(sc), np.exp(sc - sc.max(axis=1, keepdims=True)), 0.0)
    return ((e / e.sum(axis=1, keepdims=True)) @ v.astype(np.float64)).astype(np.result_type(q, v))


# ---------------------------------------------------------------------------
# neuron-sparse MLP (sf/neuron_ops.py:22-95)


def n_blocks(d_ff: int, blk: int) -> int:
    return -(-d_ff // blk)


def active_columns(mask, d_ff: int, blk: int):
    """sf/neuron_ops.py:59-72: ascending active blocks and their hidden columns."""
    mask = np.asarray(mask, dtype=bool)
    if mask.shape != (n_blocks(d_ff, blk),):
        raise MaskError(f"mask length {mask.shape} != n_blk ({n_blocks(d_ff, blk)},)")
    active = np.flatnonzero(mask)
    cols = (active[:, None] * blk + np.arange(blk)[None, :]).reshape(-1)
    cols = cols[cols < d_ff]
    return tuple(int(b) for b in active), cols


def neuron_matmul_fwd1(x, w1, mask, blk):
    """sf/neuron_ops.py:75-82: x @ W1[:, cols] (w1 is [d, d_ff])."""
    _, cols = active_columns(mask, w1.shape[1], blk)
    return (x @ w1[:, cols] if cols.size else np.zeros((x.shape[0], 0), x.dtype)), cols


def neuron_matmul_fwd2(values, w2, cols):
    """sf/neuron_ops.py:85-95: packed hidden @ W2[cols, :]."""
    if cols.size == 0:
        return np.zeros((values.shape[0], w2.shape[1]), dtype=values.dtype)
    return values @ w2[cols, :]


# ---------------------------------------------------------------------------
# model with frozen backbone + PEFT (sf/model.py:28-472) and backward (sf/autograd.py)

LORA_SHAPES = {"wq": "attn", "wk": "attn", "wv": "attn", "wo": "attn", "w1": "mlp_in", "w2": "mlp_out"}
BIAS_NAMES = ("bq", "bk", "bv", "bo", "b1", "b2")


@dataclass(frozen=True)
class Dims:
    """sf/model.py:33-60."""

    d_model: int
    n_heads: int
    d_ff: int
    seq_len: int
    n_layers: int = 4
    vocab: int = 256
    blk_size: int = 16
    attn_blk: int = 16

    @property
    def head_dim(self):
        return self.d_model // self.n_heads

    @property
    def n_blk(self):
        return n_blocks(self.d_ff, self.blk_size)

    @property
    def n_b(self):
        return self.seq_len // self.attn_blk


@dataclass
class OModel:
    dims: Dims
    peft: str
    emb: np.ndarray
    layers: list  # list of dict of arrays; w1 is [d, d_ff]
    lnf_g: np.ndarray
    lnf_b: np.ndarray
    pool: dict
    lora: dict = field(default_factory=dict)  # (layer, target) -> {"a","b","scaling"}
    adapters: dict = field(default_factory=dict)  # (layer, sub) -> {"w_down","b_down","w_up","b_up"}
    lora_targets: tuple = ()

    def astype(self, dtype):
        import copy

        m = copy.deepcopy(self)
        for lw in m.layers:
            for k in lw:
                lw[k] = lw[k].astype(dtype)
        m.emb, m.lnf_g, m.lnf_b = m.emb.astype(dtype), m.lnf_g.astype(dtype), m.lnf_b.astype(dtype)
        for ad in list(m.lora.values()) + list(m.adapters.values()):
            for k in ad:
                if isinstance(ad[k], np.ndarray):
                    ad[k] = ad[k].astype(dtype)
        return m


def build_model(dims: Dims, seed: int, peft="lora", lora_rank=8, lora_targets=("wq", "wv", "w1", "w2"), adapter_rank=8, init_scale=0.02) -> OModel:
    """sf/model.py:174-231 — same PCG64 draw order, so weights are identical."""
    if peft not in ("lora", "adapter", "bitfit"):
        raise ValueError(f"unknown peft method {peft!r}")
    rng = make_rng(seed)
    d, f = dims.d_model, dims.d_ff
    z = lambda n: np.zeros(n, np.float32)  # noqa: E731
    layers = []
    for _ in range(dims.n_layers):
        wq, wk, wv, wo = (randn(rng, (d, d), init_scale) for _ in range(4))
        w1 = randn(rng, (d, f), init_scale)
        w2 = randn(rng, (f, d), init_scale)
        layers.append(dict(wq=wq, wk=wk, wv=wv, wo=wo, bq=z(d), bk=z(d), bv=z(d), bo=z(d), w1=w1, w2=w2, b1=z(f), b2=z(d),
                           ln1_g=np.ones(d, np.float32), ln1_b=z(d), ln2_g=np.ones(d, np.float32), ln2_b=z(d)))
    emb = randn(rng, (dims.vocab, d), init_scale)
    m = OModel(dims, peft, emb, layers, np.ones(d, np.float32), z(d), build_pool(dims.n_b),
               lora_targets=tuple(lora_targets) if peft == "lora" else ())
    if peft == "lora":
        shapes = {"attn": (d, d), "mlp_in": (d, f), "mlp_out": (f, d)}
        for i in range(dims.n_layers):
            for t in m.lora_targets:
                di, do = shapes[LORA_SHAPES[t]]
                m.lora[(i, t)] = {"a": randn(rng, (di, lora_rank), init_scale), "b": np.zeros((lora_rank, do), np.float32), "scaling": 1.0}
    elif peft == "adapter":
        for i in range(dims.n_layers):
            for sub in ("attn", "mlp"):
                m.adapters[(i, sub)] = {"w_down": randn(rng, (d, adapter_rank), init_scale), "b_down": z(adapter_rank),
                                        "w_up": np.zeros((adapter_rank, d), np.float32), "b_up": z(d)}
    return m


def trainable_params(m: OModel) -> dict:
    """sf/model.py:234-249 (names and order)."""
    out = {}
    if m.peft == "lora":
        for (i, t), ad in sorted(m.lora.items()):
            out[f"layers.{i}.{t}.lora_a"] = ad["a"]
            out[f"layers.{i}.{t}.lora_b"] = ad["b"]
    elif m.peft == "adapter":
        for (i, sub), ad in sorted(m.adapters.items()):
            for k in ("w_down", "b_down", "w_up", "b_up"):
                out[f"layers.{i}.{sub}_adapter.{k}"] = ad[k]
    else:
        for i, lw in enumerate(m.layers):
            for b in BIAS_NAMES:
                out[f"layers.{i}.{b}"] = lw[b]
    return out


def lora_linear_forward(x, w, bias, ad):
    """sf/model.py:292-304."""
    z = x @ w
    ax = None
    if ad is not None:
        ax = x @ ad["a"]
        z = z + ad["scaling"] * (ax @ ad["b"])
    if bias is not None:
        z = z + bias
    return z, {"x": x, "ax": ax}


def layernorm_forward(x, g, b, eps=1e-5):
    """sf/model.py:307-312."""
    mu = x.mean(axis=1, keepdims=True)
    inv = 1.0 / np.sqrt(x.var(axis=1, keepdims=True) + eps)
    xh = (x - mu) * inv
    return xh * g + b, {"xhat": xh, "inv_std": inv, "gamma": g}


def layernorm_backward(dy, c):
    """sf/autograd.py:61-66."""
    g = dy * c["gamma"]
    xh = c["xhat"]
    return c["inv_std"] * (g - g.mean(axis=1, keepdims=True) - xh * (g * xh).mean(axis=1, keepdims=True))


def adapter_forward(x, ad):
    """sf/model.py:315-319."""
    z = x @ ad["w_down"] + ad["b_down"]
    h = np.maximum(z, 0)
    return x + h @ ad["w_up"] + ad["b_up"], {"x": x, "z": z, "h": h}


def _acc(grads, name, val):
    grads[name] = grads[name] + val if name in grads else val


def adapter_backward(dy, ad, c, grads, prefix):
    """sf/autograd.py:69-75."""
    _acc(grads, f"{prefix}.w_up", c["h"].T @ dy)
    _acc(grads, f"{prefix}.b_up", dy.sum(axis=0))
    dh = (dy @ ad["w_up"].T) * (c["z"] > 0)
    _acc(grads, f"{prefix}.w_down", c["x"].T @ dh)
    _acc(grads, f"{prefix}.b_down", dh.sum(axis=0))
    return dy + dh @ ad["w_down"].T


def lora_linear_backward(dz, w, ad, c, grads, prefix, bias_name):
    """sf/autograd.py:48-58."""
    dx = dz @ w.T
    if ad is not None:
        dax = dz @ ad["b"].T * ad["scaling"]
        _acc(grads, f"{prefix}.lora_a", c["x"].T @ dax)
        _acc(grads, f"{prefix}.lora_b", ad["scaling"] * (c["ax"].T @ dz))
        dx = dx + dax @ ad["a"].T
    if bias_name is not None:
        _acc(grads, bias_name, dz.sum(axis=0))
    return dx


def mha_forward(x, lw, lora, head_patterns, pool, dims: Dims):
    """sf/model.py:322-360 (non-causal; per-head SDD -> sparse softmax -> DSD)."""
    if len(head_patterns) != dims.n_heads:
        raise ShapeError(f"expected {dims.n_heads} head patterns, got {len(head_patterns)}")
    for pid in head_patterns:
        if pid not in pool:
            raise PatternError(f"pattern id {pid!r} not in pool")
    q, cq = lora_linear_forward(x, lw["wq"], lw["bq"], lora.get("wq"))
    k, ck = lora_linear_forward(x, lw["wk"], lw["bk"], lora.get("wk"))
    v, cv = lora_linear_forward(x, lw["wv"], lw["bv"], lora.get("wv"))
    hd, blk, n_b = dims.head_dim, dims.attn_blk, dims.n_b
    scale = 1.0 / np.sqrt(hd)
    heads = np.empty_like(q)
    probs = []
    for h, pid in enumerate(head_patterns):
        sl = slice(h * hd, (h + 1) * hd)
        coords = pool[pid]
        p = sparse_softmax(sdd(q[:, sl], k[:, sl], coords, blk, scale), coords, n_b)
        probs.append(p)
        heads[:, sl] = dsd(p, v[:, sl], coords, n_b)
    out, co = lora_linear_forward(heads, lw["wo"], lw["bo"], lora.get("wo"))
    return out, {"q": q, "k": k, "v": v, "heads_out": heads, "probs": probs, "patterns": list(head_patterns),
                 "cq": cq, "ck": ck, "cv": cv, "co": co}


def mha_backward(d_out, c, lw, lora, pool, dims: Dims, grads, prefix="", bitfit=False):
    """sf/autograd.py:127-162."""
    dh = lora_linear_backward(d_out, lw["wo"], lora.get("wo"), c["co"], grads, f"{prefix}wo", f"{prefix}bo" if bitfit else None)
    q, k, v = c["q"], c["k"], c["v"]
    hd, blk, n_b = dims.head_dim, dims.attn_blk, dims.n_b
    scale = 1.0 / np.sqrt(hd)
    dq, dk, dv = np.zeros_like(q), np.zeros_like(k), np.zeros_like(v)
    for h, pid in enumerate(c["patterns"]):
        sl = slice(h * hd, (h + 1) * hd)
        coords = pool[pid]
        p = c["probs"][h]
        db, dv[:, sl] = dsd_backward(p, v[:, sl], dh[:, sl], coords, n_b)
        ds = sparse_softmax_backward(p, db, coords, n_b)
        dq[:, sl], dk[:, sl] = sdd_backward(ds, q[:, sl], k[:, sl], coords, blk, scale)
    dx = lora_linear_backward(dq, lw["wq"], lora.get("wq"), c["cq"], grads, f"{prefix}wq", f"{prefix}bq" if bitfit else None)
    dx = dx + lora_linear_backward(dk, lw["wk"], lora.get("wk"), c["ck"], grads, f"{prefix}wk", f"{prefix}bk" if bitfit else None)
    dx = dx + lora_linear_backward(dv, lw["wv"], lora.get("wv"), c["cv"], grads, f"{prefix}wv", f"{prefix}bv" if bitfit else None)
    return dx


def mlp_forward(x, lw, lora, neuron_mask, dims: Dims):
    """sf/model.py:363-400."""
    values, cols = neuron_matmul_fwd1(x, lw["w1"], neuron_mask, dims.blk_size)
    z = values + lw["b1"][cols]
    ad1, ax1 = lora.get("w1"), None
    if ad1 is not None and cols.size:
        ax1 = x @ ad1["a"]
        z = z + ad1["scaling"] * (ax1 @ ad1["b"][:, cols])
    a = np.maximum(z, 0)
    out = neuron_matmul_fwd2(a, lw["w2"], cols) + lw["b2"]
    ad2, ax2 = lora.get("w2"), None
    if ad2 is not None and cols.size:
        ax2 = a @ ad2["a"][cols, :]
        out = out + ad2["scaling"] * (ax2 @ ad2["b"])
    return out, {"x": x, "z": z, "a": a, "cols": cols, "mask": np.asarray(neuron_mask, bool), "ax1": ax1, "ax2": ax2}


def mlp_backward(d_out, c, lw, lora, neuron_mask, dims: Dims, grads, prefix="", bitfit=False):
    """sf/autograd.py:78-124."""
    if not np.array_equal(c["mask"], np.asarray(neuron_mask, bool)):
        raise GradientError("cache was produced with a different neuron mask")
    cols, x, z, a = c["cols"], c["x"], c["z"], c["a"]
    if bitfit:
        _acc(grads, f"{prefix}b2", d_out.sum(axis=0))
    da = d_out @ lw["w2"][cols, :].T if cols.size else np.zeros_like(a)
    ad2 = lora.get("w2")
    if ad2 is not None and cols.size:
        dax2 = d_out @ ad2["b"].T * ad2["scaling"]
        _acc(grads, f"{prefix}w2.lora_b", ad2["scaling"] * (c["ax2"].T @ d_out))
        g = np.zeros_like(ad2["a"])
        g[cols, :] = a.T @ dax2
        _acc(grads, f"{prefix}w2.lora_a", g)
        da = da + dax2 @ ad2["a"][cols, :].T
    dz = da * (z > 0)
    if bitfit:
        g = np.zeros_like(lw["b1"])
        if cols.size:
            g[cols] = dz.sum(axis=0)
        _acc(grads, f"{prefix}b1", g)
    dx = dz @ lw["w1"][:, cols].T if cols.size else np.zeros_like(x)
    ad1 = lora.get("w1")
    if ad1 is not None:
        gb = np.zeros_like(ad1["b"])
        if cols.size:
            gb[:, cols] = ad1["scaling"] * (c["ax1"].T @ dz)
            dax1 = dz @ ad1["b"][:, cols].T * ad1["scaling"]
            _acc(grads, f"{prefix}w1.lora_a", x.T @ dax1)
            dx = dx + dax1 @ ad1["a"].T
        else:
            _acc(grads, f"{prefix}w1.lora_a", np.zeros_like(ad1["a"]))
        _acc(grads, f"{prefix}w1.lora_b", gb)
    return dx


def _layer_lora(m: OModel, i: int) -> dict:
    return {t: m.lora[(i, t)] for t in m.lora_targets} if m.peft == "lora" else {}


def block_forward(x, m: OModel, i: int, masks):
    """sf/model.py:403-433. `masks` = (head_patterns, neuron_mask) or a provider."""
    lw, lora = m.layers[i], _layer_lora(m, i)
    h1, c1 = layernorm_forward(x, lw["ln1_g"], lw["ln1_b"])
    pats = masks[0] if isinstance(masks, tuple) else masks.attn_patterns(i, h1)
    att, ca = mha_forward(h1, lw, lora, pats, m.pool, m.dims)
    caa = None
    if m.peft == "adapter":
        att, caa = adapter_forward(att, m.adapters[(i, "attn")])
    y = x + att
    h2, c2 = layernorm_forward(y, lw["ln2_g"], lw["ln2_b"])
    nm = masks[1] if isinstance(masks, tuple) else masks.mlp_mask(i, h2)
    mo, cm = mlp_forward(h2, lw, lora, nm, m.dims)
    cma = None
    if m.peft == "adapter":
        mo, cma = adapter_forward(mo, m.adapters[(i, "mlp")])
    return y + mo, {"ln1": c1, "attn": ca, "attn_ad": caa, "ln2": c2, "mlp": cm, "mlp_ad": cma,
                    "masks": (list(pats), np.asarray(nm, bool))}


def block_backward(d_out, m: OModel, i: int, c, grads):
    """sf/autograd.py:165-181."""
    lw, lora, bitfit, prefix = m.layers[i], _layer_lora(m, i), m.peft == "bitfit", f"layers.{i}."
    dm = d_out
    if m.peft == "adapter":
        dm = adapter_backward(d_out, m.adapters[(i, "mlp")], c["mlp_ad"], grads, f"{prefix}mlp_adapter")
    dh2 = mlp_backward(dm, c["mlp"], lw, lora, c["masks"][1], m.dims, grads, prefix, bitfit)
    dy = d_out + layernorm_backward(dh2, c["ln2"])
    da = dy
    if m.peft == "adapter":
        da = adapter_backward(dy, m.adapters[(i, "attn")], c["attn_ad"], grads, f"{prefix}attn_adapter")
    dh1 = mha_backward(da, c["attn"], lw, lora, m.pool, m.dims, grads, prefix, bitfit)
    return dy + layernorm_backward(dh1, c["ln1"])


def model_forward(m: OModel, tokens, masks):
    """sf/model.py:436-451 (no positional embedding; tied unembedding)."""
    if tokens.max() >= m.dims.vocab or tokens.min() < 0:
        raise ValueError("token id out of vocab range")
    h = m.emb[tokens]
    caches = []
    for i in range(m.dims.n_layers):
        lm = masks[i] if isinstance(masks, list) else masks
        h, c = block_forward(h, m, i, lm)
        caches.append(c)
    hf, cf = layernorm_forward(h, m.lnf_g, m.lnf_b)
    return hf @ m.emb.T, {"blocks": caches, "lnf": cf}


def loss_forward(logits, targets) -> float:
    """sf/model.py:454-462."""
    sh = logits - logits.max(axis=1, keepdims=True)
    return float(np.mean(np.log(np.exp(sh).sum(axis=1)) - sh[np.arange(len(targets)), targets]))


def loss_backward(logits, targets):
    """sf/model.py:465-472."""
    e = np.exp(logits - logits.max(axis=1, keepdims=True))
    g = e / e.sum(axis=1, keepdims=True)
    g[np.arange(len(targets)), targets] -= 1.0
    return g / len(targets)


def model_backward(m: OModel, cache, d_logits):
    """sf/autograd.py:184-196."""
    grads = {}
    dh = layernorm_backward(d_logits @ m.emb, cache["lnf"])
    for i in reversed(range(m.dims.n_layers)):
        dh = block_backward(dh, m, i, cache["blocks"][i], grads)
    for name, p in trainable_params(m).items():
        if name not in grads:
            grads[name] = np.zeros_like(p)
    return grads


def optimizer_step(params: dict, mom: dict, vel: dict, step: int, grads: dict, lr, betas=(0.9, 0.999), eps=1e-8) -> int:
    """sf/autograd.py:203-225 — Adam with float64 moments, in place; returns new step."""
    b1, b2 = betas
    t = step + 1
    for name, p in params.items():
        g = grads[name].astype(np.float64)
        mom[name] = b1 * mom.get(name, 0.0) + (1 - b1) * g
        vel[name] = b2 * vel.get(name, 0.0) + (1 - b2) * g * g
        p -= (lr * (mom[name] / (1 - b1**t)) / (np.sqrt(vel[name] / (1 - b2**t)) + eps)).astype(p.dtype)
    return t


class PredictedProvider:
    """sf/harness.py:193-211: per-item attention patterns and MLP masks from
    predictor weights (the fine-tune loop calls it with a one-item batch)."""

    def __init__(self, m: OModel, attn_params: list, mlp_params: list, cfg: PredictorConfig):
        self.m, self.attn, self.mlp, self.cfg = m, attn_params, mlp_params, cfg

    def attn_patterns(self, i, h):
        return predict_attention_patterns([h], self.attn[i], self.m.pool, self.cfg)

    def mlp_mask(self, i, h):
        return predict_mlp_mask([approx_mlp_scores(h, self.mlp[i])], self.cfg.mlp_threshold)


def finetune_step(m: OModel, batch_tokens, provider, params, mom, vel, step, lr):
    """One step of sf/harness.py:396-417 (per-item fwd/bwd, grads mean, Adam)."""
    gsum, losses = {}, []
    for seq in batch_tokens:
        tok, tgt = seq[:-1], seq[1:]
        logits, cache = model_forward(m, tok, provider)
        losses.append(loss_forward(logits, tgt))
        g = model_backward(m, cache, loss_backward(logits, tgt))
        for k, v in g.items():
            gsum[k] = gsum.get(k, 0) + v
    gmean = {k: v / len(batch_tokens) for k, v in gsum.items()}
    step = optimizer_step(params, mom, vel, step, gmean, lr)
    return float(np.mean(losses)), gmean, step
