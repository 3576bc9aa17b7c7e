"""Mask providers and the fine-tune step (drop-in for the hot-path half of
sf/harness.py:122-244 and the inner loop of run_finetune, sf/harness.py:396-427).

Providers implement the reference protocol `attn_patterns(layer, h)` /
`mlp_mask(layer, h)`. The predicted provider returns device-resident results
(pool indices [B, H] and compacted neuron index lists) so a step never
synchronises the host; it also asks block_forward for the LayerNorm-fused
downsampled rows (`fused_downsample`). Prediction time is measured with CUDA
events on the current stream (the reference uses perf_counter around the
same calls) and reported without a sync until `elapsed_ns` is read.
"""

from __future__ import annotations

import numpy as np
import torch

from . import autograd, exposer as EX, model as M, predictor as P
from .errors import ConfigError

MODES = ("dense", "shadowy", "exposer-oracle", "predicted", "random")


class _TimedProvider:
    def __init__(self):
        self._events: list = []
        self.timing = True

    def _timed(self, fn, *a, **k):
        if not self.timing:
            return fn(*a, **k)
        st = torch.cuda.Event(enable_timing=True)
        en = torch.cuda.Event(enable_timing=True)
        st.record()
        out = fn(*a, **k)
        en.record()
        self._events.append((st, en))
        return out

    @property
    def elapsed_ns(self) -> int:
        torch.cuda.synchronize()
        return int(sum(s.elapsed_time(e) for s, e in self._events) * 1e6)

    def reset_timing(self):
        self._events.clear()

    def attn_patterns(self, layer: int, h, x_small=None):
        return self._timed(self._attn, layer, h, x_small)

    def mlp_mask(self, layer: int, h):
        return self._timed(self._mlp, layer, h)


class DenseProvider(_TimedProvider):
    """sf/harness.py:145-154."""

    def __init__(self, model: M.Model):
        super().__init__()
        self.model = model

    def _attn(self, layer, h, x_small=None):
        return ["dense"] * self.model.dims.n_heads

    def _mlp(self, layer, h):
        return np.ones(self.model.dims.n_blk, dtype=bool)


class PredictedProvider(_TimedProvider):
    """sf/harness.py:193-211 on the fused mask-build kernels. scope='item' gives the
    fine-tune loop's per-sequence masks; scope='batch' ORs over the batch (sf/predictor.py:105-136)."""

    fused_downsample = True

    def __init__(self, model: M.Model, predictors: dict, cfg: P.PredictorTrainConfig | None = None, counter=None,
                 scope: str = "item"):
        super().__init__()
        if scope not in ("item", "batch"):
            raise ConfigError(f"unknown mask scope {scope!r}")
        self.model, self.predictors, self.counter = model, predictors, counter
        self.pcfg = cfg or P.PredictorTrainConfig()
        self.scope_batch = scope == "batch"
        self.last_scores = {}

    def _attn(self, layer, h, x_small=None):
        B, s, d = h.shape
        if x_small is None:
            x_small, m = P.x_small_of(h)
        else:
            m = x_small.shape[0] // B
        params = self.predictors["attn"][layer]
        idx, _ = P.attn_pattern_idx(x_small, B, m, params, self.model.dpool, self.model.dims.n_b, self.pcfg,
                                    scope_batch=self.scope_batch)
        if self.counter is not None:
            self.counter.add(B * len(params.wq_hat) * (2 * m * d * params.rank + m * m * params.rank))
        return idx

    def _mlp(self, layer, h):
        B, s, d = h.shape
        params = self.predictors["mlp"][layer]
        nm, _ = P.mlp_masks(h.reshape(B * s, d), B, s, params, self.pcfg.mlp_threshold, self.model.dims.blk_size,
                            terms=self.pcfg.score_terms,
                            scope_batch=self.scope_batch)
        if self.counter is not None:
            self.counter.add(B * (s * d * self.model.dims.n_blk + s))
        return nm


class OracleProvider(_TimedProvider):
    """Ground-truth masks from the exact dense computation (sf/harness.py:157-176); verification
    mode. Per item: exact block masses of every head -> coverage-selected pool pattern; exact
    MLP pre-activation -> block importance -> theta filter. Device-resident like PredictedProvider."""

    def __init__(self, model: M.Model, theta: float, tau: float):
        super().__init__()
        if not (0 <= theta <= 1):
            raise ConfigError(f"theta must be in [0, 1], got {theta}")
        if not (0 < tau <= 1):
            raise ConfigError(f"coverage tau must be in (0, 1], got {tau}")
        self.model, self.theta, self.tau = model, theta, tau

    _head_sum = False

    def _attn(self, layer, h, x_small=None):
        B, s, _ = h.shape
        dims = self.model.dims
        mass = EX.exact_block_mass(EX.exact_qk(h, self.model.weights.layers[layer]), B, s, dims.n_heads, dims.n_b)
        return EX.select_by_coverage(mass, self.model.dpool, self.tau, head_sum=self._head_sum)

    def _mlp(self, layer, h):
        B, s, _ = h.shape
        m = self.model
        ad = m.lora.get((layer, "w1")) if m.peft_method == "lora" else None
        z = EX.mlp_preactivation(h, m.weights.layers[layer], ad)
        imp = EX.block_importance(z, B, s, m.dims.blk_size)
        return EX.filter_neuron_blocks(imp, self.theta, m.dims.blk_size)


class ShadowyProvider(OracleProvider):
    """One attention pattern for all heads from the head-summed block masses; MLP keeps every
    block any token activates (theta = 0) — sf/harness.py:179-190."""

    _head_sum = True

    def __init__(self, model: M.Model, tau: float):
        super().__init__(model, theta=0.0, tau=tau)


def make_provider(cfg, model: M.Model, predictors=None, counter=None, *, theta: float = 0.1, tau: float = 0.95,
                  seed: int = 0, pcfg=None, scope: str = "item") -> _TimedProvider:
    """sf/harness.py:233-244. `cfg` is the reference's RunConfig (or any object with its `mode`, `theta`,
    `tau`, `seed`, `tau_pred`, `attn_threshold_frac` and `mlp_threshold` fields), so a reference call
    make_provider(cfg, model, predictors, counter) drops in unchanged; a bare mode string with keyword
    overrides is also accepted. Unknown modes fall through to RandomProvider, as in the reference."""
    if isinstance(cfg, str):
        mode = cfg
    else:
        mode = cfg.mode
        theta, tau, seed = cfg.theta, cfg.tau, cfg.seed
        if pcfg is None and hasattr(cfg, "tau_pred"):
            pcfg = P.PredictorTrainConfig(attn_threshold_frac=cfg.attn_threshold_frac, mlp_threshold=cfg.mlp_threshold,
                                          tau_pred=cfg.tau_pred)
    if mode == "dense":
        return DenseProvider(model)
    if mode == "shadowy":
        return ShadowyProvider(model, tau)
    if mode == "exposer-oracle":
        return OracleProvider(model, theta, tau)
    if mode == "predicted":
        if predictors is None:
            raise ConfigError("mode=predicted requires trained predictors")
        return PredictedProvider(model, predictors, pcfg, counter=counter, scope=scope)
    return RandomProvider(model, seed=seed + 10_000)


class RandomProvider(_TimedProvider):
    """Seeded random patterns (sf/harness.py:214-230), the convergence-ablation baseline."""

    def __init__(self, model: M.Model, seed: int):
        super().__init__()
        self.model = model
        self.rng = np.random.Generator(np.random.PCG64(seed))
        self.pattern_ids = [p for p in model.pool if p != "dense"]

    def _attn(self, layer, h, x_small=None):
        return [self.pattern_ids[self.rng.integers(len(self.pattern_ids))] for _ in range(self.model.dims.n_heads)]

    def _mlp(self, layer, h):
        mask = self.rng.random(self.model.dims.n_blk) < 0.5
        if not mask.any():
            mask[self.rng.integers(len(mask))] = True
        return mask


def finetune_step(model: M.Model, state: M.PeftState, batch_tokens, provider, lr: float, grad_hook=None) -> dict:
    """One optimiser step of run_finetune (sf/harness.py:396-417) over a batch [B, s+1]:
    per-item masks, mean loss, grads summed over items then / B, Adam (float64 moments).
    `grad_hook(flat)` runs before the update on the flat fp32 mean-gradient buffer (state.flat's layout)
    and reduces it in place (the data-parallel all-reduce, dp.make_grad_hook)."""
    tok = torch.as_tensor(np.asarray(batch_tokens) if not torch.is_tensor(batch_tokens) else batch_tokens)
    tok = tok.to(model.device, torch.int64)
    inp, tgt = tok[:, :-1], tok[:, 1:]
    logits, cache = M.model_forward(model, inp, provider)
    loss = M.loss_forward(logits, tgt)
    grads = autograd.model_backward(model, cache, M.loss_backward(logits, tgt))
    B = tok.shape[0]
    mean = {n: g / B for n, g in grads.items()}
    if grad_hook is not None:
        # same contract as FinetuneEngine: the hook reduces the flat fp32 mean-gradient buffer (laid out like
        # state.flat) in place, e.g. dp.make_grad_hook's all-reduce; its return value is ignored
        flat = torch.empty_like(state.flat)
        for n, p in state.params.items():
            off = (p.data_ptr() - state.flat.data_ptr()) // 4
            flat[off : off + p.numel()] = mean[n].reshape(-1)
        grad_hook(flat)
        for n, p in state.params.items():
            off = (p.data_ptr() - state.flat.data_ptr()) // 4
            mean[n] = flat[off : off + p.numel()].view(p.shape)
    autograd.optimizer_step(state, mean, lr)
    if not np.isfinite(loss):
        raise FloatingPointError(f"non-finite loss {loss}")
    return {"loss": loss, "grads": mean, "masks": [c["masks"] for c in cache["blocks"]]}
