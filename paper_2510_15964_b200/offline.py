"""Offline predictor pipeline on the GPU: trace collection, predictor training and the
`.tnsc` predictor files (sf/harness.py:251-371, sf/predictor.py:171-298, sf/containers.py).

Trace collection runs the dense forward once per batch of sequences on the device and
keeps, per layer, what training reads:

* attention — the downsampled rows of the attention input (`x_attn_ds`, m = ceil(sqrt(s))
  rows, sf/predictor.py:62-71) and the downsampled exact raw scores per head (`raw_ds.h*`,
  m x m float64, the only part of the s x s scores train_attn_predictor uses,
  sf/predictor.py:222-224) instead of the full probs + raw (2 H s^2 values per layer);
* MLP — the full input `x_mlp` and the per-token block-activity bits of the exact
  pre-activation (`mlp_active`, 64 blocks per int64 word; mlp_truth_labels,
  sf/predictor.py:251-259) instead of z [s, d_ff].

`full=True` writes the reference's own keys (x_attn, x_mlp, z, probs.h*, raw.h*) so the
file is a drop-in for sf/harness.py:load_traces; `load_traces` reads either form.

Training keeps the reference's objectives and optimiser (MSE distillation of the
downsampled scores; recall-weighted logistic regression; Adam, float64 moments) with every
head of a layer trained in one batched pass: projections and scores as batched fp32 GEMMs,
the score-gradient contractions in float64 (as the reference's float64 broadcasting makes
them), the weighted logistic loss and its gradient in one kernel (lx_weighted_bce), truth
labels from lx_block_activity, the update from lx_adam_step. Input noise is drawn from a
seeded torch generator on the device (the reference draws NumPy noise per head/epoch);
with noise_std = 0 the result matches the reference to float rounding.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _abi, exposer as EX, model as M
from .predictor import (AttnPredictorParams, MlpPredictorParams, PredictorTrainConfig, approx_mlp_scores,
                        attn_pattern_idx, binarize_scores, downsample_indices, eval_recall_precision, upsample_mask)
from .tnsc import load_tensors, save_tensors


# ---------------------------------------------------------------------------- seeded init
def make_rng(seed: int) -> np.random.Generator:
    """sf/tensor_core.py:19-21."""
    return np.random.Generator(np.random.PCG64(seed))


def randn(rng: np.random.Generator, shape, scale: float) -> np.ndarray:
    """sf/tensor_core.py:24-28."""
    if scale <= 0:
        raise ValueError(f"scale must be > 0, got {scale}")
    return (rng.standard_normal(shape) * scale).astype(np.float32)


def init_attn_predictor(d: int, n_heads: int, rank: int | None = None, seed: int = 0) -> AttnPredictorParams:
    """sf/predictor.py:194-201 (same draws, same order)."""
    rank = rank if rank is not None else max(4, d // 16)
    rng = make_rng(seed)
    wq = [randn(rng, (d, rank), 0.1) for _ in range(n_heads)]
    wk = [randn(rng, (d, rank), 0.1) for _ in range(n_heads)]
    return AttnPredictorParams(wq_hat=wq, wk_hat=wk)


def init_mlp_predictor(d: int, n_blk: int, seed: int = 0) -> MlpPredictorParams:
    """sf/predictor.py:204-206."""
    return MlpPredictorParams(wa_hat=randn(make_rng(seed), (d, n_blk), 0.1))


# ---------------------------------------------------------------------------- block activity bits
def mlp_truth_labels(z: torch.Tensor, blk: int) -> torch.Tensor:
    """mlp_truth_labels (sf/predictor.py:251-259) on the device: int32 bit words [rows, ceil(n_blk/32)]."""
    z = z.float()
    if z.stride(1) != 1:
        z = z.contiguous()
    rows, n_cols = z.shape
    n_blk = -(-n_cols // blk)
    bits = torch.empty(rows, (n_blk + 31) // 32, dtype=torch.int32, device=z.device)
    _abi.call("lx_block_activity", z.data_ptr(), z.stride(0), rows, n_cols, blk, bits.data_ptr(),
              _abi.stream_handle(z.device))
    return bits


def bits_to_bool(bits, n_blk: int) -> torch.Tensor:
    """[rows, words32] int32 -> bool [rows, n_blk]."""
    bits = torch.as_tensor(bits)
    sh = torch.arange(32, device=bits.device, dtype=torch.int32)
    return (((bits[:, :, None] >> sh) & 1).reshape(bits.shape[0], -1)[:, :n_blk]).bool()


def _words32_to_64(bits32: np.ndarray) -> np.ndarray:
    b = np.ascontiguousarray(bits32, dtype=np.int32)
    if b.shape[1] % 2:
        b = np.concatenate([b, np.zeros((b.shape[0], 1), np.int32)], 1)
    return b.view(np.int64)


def _words64_to_32(bits64: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(bits64, dtype=np.int64).view(np.int32)


# ---------------------------------------------------------------------------- traces
@torch.no_grad()
def collect_traces(model: M.Model, corpus, path=None, batch: int = 8, full: bool = False) -> dict:
    """run_collect_traces (sf/harness.py:249-265) on the device: dense forward over `corpus`
    ([n, s] tokens) in batches; returns (and writes to `path` if given) the trace tensors.

    full=False (default) writes the compact schema (x_attn_ds / mlp_active / raw_ds): what the trainers
    read, ~35x smaller. It is ONE-WAY: `load_traces` here reads it, the reference's load_traces
    (sf/harness.py:268-285) does not. Pass full=True to write the reference's own keys for a trace file the
    reference will read."""
    corpus = np.asarray(corpus)
    n, s = corpus.shape
    dims = model.dims
    H, d, hd = dims.n_heads, dims.d_model, dims.d_model // dims.n_heads
    idx = torch.as_tensor(downsample_indices(s), device=model.device)
    m = idx.numel()
    scale = 1.0 / float(np.sqrt(hd))
    out: dict[str, np.ndarray] = {} if full else {"meta.n_blk": np.array([dims.n_blk], np.int64)}
    for b0 in range(0, n, batch):
        tok = torch.as_tensor(corpus[b0 : b0 + batch], dtype=torch.int64, device=model.device)
        B = tok.shape[0]
        rec = EX._Recorder(model)
        M.model_forward(model, tok, rec)
        for layer in range(dims.n_layers):
            lw = model.weights.layers[layer]
            ha, hm = rec.h_attn[layer], rec.h_mlp[layer]  # bf16 [B, s, d]
            xs = ha[:, idx]  # [B, m, d]
            qk = EX.exact_qk(xs, lw).view(B, m, 2, H, hd)
            q, k = qk[:, :, 0].permute(0, 2, 1, 3), qk[:, :, 1].permute(0, 2, 1, 3)  # [B, H, m, hd]
            raw_ds = (q @ k.transpose(-1, -2)).double() * scale  # float32 scores, float64 scale (sf/exposer.py:56)
            ad = model.lora.get((layer, "w1")) if model.peft_method == "lora" else None
            z = EX.mlp_preactivation(hm, lw, ad)  # fp32 [B*s, d_ff]
            bits = mlp_truth_labels(z, dims.blk_size).view(B, s, -1).cpu().numpy()
            xs_h, hm_h, raw_h = xs.float().cpu().numpy(), hm.float().cpu().numpy(), raw_ds.cpu().numpy()
            if full:
                qkf = EX.exact_qk(ha, lw).view(B, s, 2, H, hd)
                qf, kf = qkf[:, :, 0].permute(0, 2, 1, 3), qkf[:, :, 1].permute(0, 2, 1, 3)
                raw_f = (qf @ kf.transpose(-1, -2)).double() * scale
                probs_f = torch.softmax(raw_f, dim=-1).cpu().numpy()
                raw_f = raw_f.cpu().numpy()
                ha_h = ha.float().cpu().numpy()
                z_h = z.view(B, s, -1).cpu().numpy()
            for j in range(B):
                base = f"trace{b0 + j}.layer{layer}"
                out[f"{base}.x_mlp"] = hm_h[j]
                if full:
                    out[f"{base}.x_attn"] = ha_h[j]
                    out[f"{base}.z"] = z_h[j]
                    for h in range(H):
                        out[f"{base}.probs.h{h}"] = probs_f[j, h]
                        out[f"{base}.raw.h{h}"] = raw_f[j, h]
                else:
                    out[f"{base}.x_attn_ds"] = xs_h[j]
                    out[f"{base}.mlp_active"] = _words32_to_64(bits[j])
                    for h in range(H):
                        out[f"{base}.raw_ds.h{h}"] = raw_h[j, h]
    if path is not None:
        save_tensors(path, out)
    return out


def load_traces(src, n_layers: int, n_heads: int, blk: int, device="cuda") -> list[list[dict]]:
    """load_traces (sf/harness.py:268-284) for either trace form: per trace, per layer
    {"x_attn_ds" [m, d], "raw_ds" [H x (m, m)], "x_mlp" [s, d], "active_bits" int32 words [s, ceil(n_blk/32)]}
    (the full form's z is reduced to activity bits on `device`)."""
    tensors = src if isinstance(src, dict) else load_tensors(src)[0]
    n_traces = 1 + max(int(k.split(".")[0][5:]) for k in tensors if k.startswith("trace"))
    traces = []
    for i in range(n_traces):
        layers = []
        for layer in range(n_layers):
            base = f"trace{i}.layer{layer}"
            x_mlp = tensors[f"{base}.x_mlp"]
            if f"{base}.x_attn_ds" in tensors:
                xa = tensors[f"{base}.x_attn_ds"]
                raw = [tensors[f"{base}.raw_ds.h{h}"] for h in range(n_heads)]
                words = (int(tensors["meta.n_blk"][0]) + 31) // 32  # drop the int64 packing's pad word
                bits = torch.from_numpy(np.ascontiguousarray(_words64_to_32(tensors[f"{base}.mlp_active"])[:, :words]))
            else:  # the reference's full form
                ids = downsample_indices(x_mlp.shape[0])
                xa = tensors[f"{base}.x_attn"][ids]
                raw = [tensors[f"{base}.raw.h{h}"][np.ix_(ids, ids)] for h in range(n_heads)]
                z = torch.from_numpy(np.ascontiguousarray(tensors[f"{base}.z"], np.float32))
                bits = mlp_truth_labels(z.to(device), blk).cpu()
            layers.append({"x_attn_ds": xa, "raw_ds": raw, "x_mlp": x_mlp, "active_bits": bits})
        traces.append(layers)
    return traces


# ---------------------------------------------------------------------------- training
def _adam(flat: torch.Tensor, grad: torch.Tensor, mom: torch.Tensor, vel: torch.Tensor, lr: float, t: int) -> None:
    _abi.call("lx_adam_step", flat.data_ptr(), grad.data_ptr(), mom.data_ptr(), vel.data_ptr(), flat.numel(), float(lr),
              0.9, 0.999, 1e-8, int(t), _abi.stream_handle(flat.device))


def train_attn_predictor(x_ds, raw_ds, params: AttnPredictorParams, cfg: PredictorTrainConfig, seed: int = 0,
                         device="cuda") -> float:
    """train_attn_predictor (sf/predictor.py:209-248), every head at once. x_ds: per trace the
    downsampled rows [m, d]; raw_ds: per trace, per head the m x m exact raw scores. Updates
    params in place; returns the mean over heads of the last epoch's loss."""
    if not len(x_ds):
        raise ValueError("no traces")
    dev = torch.device(device)
    X = torch.as_tensor(np.stack([np.asarray(x, np.float32) for x in x_ds]), device=dev)  # [n, m, d]
    n, m, d = X.shape
    H, r = len(params.wq_hat), params.rank
    T = torch.as_tensor(np.stack([np.stack([np.asarray(raw_ds[i][h], np.float64) for i in range(n)]) for h in range(H)]),
                        device=dev)  # [H, n, m, m] float64
    flat = torch.as_tensor(np.concatenate([np.stack(params.wq_hat).ravel(), np.stack(params.wk_hat).ravel()]),
                           dtype=torch.float32, device=dev)
    wq, wk = flat[: H * d * r].view(H, d, r), flat[H * d * r :].view(H, d, r)
    mom = torch.zeros_like(flat, dtype=torch.float64)
    vel = torch.zeros_like(flat, dtype=torch.float64)
    grad = torch.empty_like(flat)
    gq, gk = grad[: H * d * r].view(H, d, r), grad[H * d * r :].view(H, d, r)
    gen = torch.Generator(device=dev).manual_seed(seed)
    Xf = X.reshape(1, n * m, d)
    losses = torch.full((H,), float("inf"), dtype=torch.float64, device=dev)
    for t in range(1, cfg.epochs + 1):
        x_in = Xf.expand(H, n * m, d)
        if cfg.noise_std > 0:  # a fresh draw per head (the reference's per-head loop)
            x_in = x_in + torch.randn(H, n * m, d, generator=gen, device=dev) * cfg.noise_std
        qh = torch.bmm(x_in, wq)  # [H, n*m, r] fp32 (x_in @ wq)
        kh = torch.bmm(x_in, wk)
        s_hat = qh.view(H, n, m, r) @ kh.view(H, n, m, r).transpose(-1, -2)  # fp32 [H, n, m, m]
        diff = s_hat.double() - T
        losses = (diff * diff).mean(dim=(1, 2, 3))
        d_s = diff * (2.0 / (n * m * m))
        xd = x_in.double().transpose(1, 2)  # [H, d, n*m]
        gq.copy_(torch.bmm(xd, (d_s @ kh.view(H, n, m, r).double()).view(H, n * m, r)))
        gk.copy_(torch.bmm(xd, (d_s.transpose(-1, -2) @ qh.view(H, n, m, r).double()).view(H, n * m, r)))
        _adam(flat, grad, mom, vel, cfg.lr, t)
    fl = losses.cpu().numpy()
    if not np.all(np.isfinite(fl)):
        raise FloatingPointError("attention predictor loss diverged")
    wq_h, wk_h = wq.cpu().numpy(), wk.cpu().numpy()
    for h in range(H):
        params.wq_hat[h] = wq_h[h].copy()
        params.wk_hat[h] = wk_h[h].copy()
    params._dev.clear()
    return float(fl.mean()) if H else 0.0


def train_mlp_predictor(x_mlp, active_bits, n_blk: int, params: MlpPredictorParams, cfg: PredictorTrainConfig,
                        seed: int = 0, device="cuda") -> float:
    """train_mlp_predictor (sf/predictor.py:262-298): recall-weighted logistic regression of the
    per-token block activity. x_mlp: per trace [s, d]; active_bits: per trace int32 words from
    mlp_truth_labels. Updates params in place; returns the last epoch's loss."""
    if not len(x_mlp):
        raise ValueError("no traces")
    dev = torch.device(device)
    X = torch.as_tensor(np.concatenate([np.asarray(x, np.float32) for x in x_mlp]), device=dev)
    Y = torch.cat([torch.as_tensor(b).to(dev, torch.int32) for b in active_bits]).contiguous()
    N, d = X.shape
    W = torch.as_tensor(np.asarray(params.wa_hat, np.float32), device=dev).contiguous()  # [d, n_blk]
    flat = W.view(-1)
    mom = torch.zeros_like(flat, dtype=torch.float64)
    vel = torch.zeros_like(flat, dtype=torch.float64)
    d_logits = torch.empty(N, n_blk, dtype=torch.float32, device=dev)
    row_loss = torch.empty(N, dtype=torch.float64, device=dev)
    gen = torch.Generator(device=dev).manual_seed(seed)
    st = _abi.stream_handle(dev)
    loss = None
    for t in range(1, cfg.epochs + 1):
        x_in = X if cfg.noise_std <= 0 else X + torch.randn(N, d, generator=gen, device=dev) * cfg.noise_std
        logits = x_in @ W  # fp32 [N, n_blk]
        _abi.call("lx_weighted_bce", logits.data_ptr(), logits.stride(0), N, n_blk, Y.data_ptr(), float(cfg.recall_weight),
                  d_logits.data_ptr(), n_blk, row_loss.data_ptr(), st)
        loss = row_loss.sum() / (N * n_blk)
        grad = (x_in.t() @ d_logits).contiguous()
        _adam(flat, grad.view(-1), mom, vel, cfg.lr, t)
    lv = float(loss) if loss is not None else float("inf")
    if not np.isfinite(lv):
        raise FloatingPointError("mlp predictor loss diverged")
    params.wa_hat = W.cpu().numpy()
    params._dev.clear()
    return lv


# ---------------------------------------------------------------------------- predictor files
def save_predictors(path, predictors: dict) -> None:
    """sf/harness.py:287-295 (same tensor names)."""
    t = {}
    for layer, p in enumerate(predictors["attn"]):
        for h in range(len(p.wq_hat)):
            t[f"layers.{layer}.attn.h{h}.wq_hat"] = np.asarray(p.wq_hat[h], np.float32)
            t[f"layers.{layer}.attn.h{h}.wk_hat"] = np.asarray(p.wk_hat[h], np.float32)
    for layer, p in enumerate(predictors["mlp"]):
        t[f"layers.{layer}.mlp.wa_hat"] = np.asarray(p.wa_hat, np.float32)
    save_tensors(path, t)


def load_predictors(path, n_layers: int, n_heads: int) -> dict:
    """sf/harness.py:298-307."""
    t, _ = load_tensors(path)
    attn = [AttnPredictorParams([t[f"layers.{i}.attn.h{h}.wq_hat"] for h in range(n_heads)],
                                [t[f"layers.{i}.attn.h{h}.wk_hat"] for h in range(n_heads)]) for i in range(n_layers)]
    mlp = [MlpPredictorParams(t[f"layers.{i}.mlp.wa_hat"]) for i in range(n_layers)]
    return {"attn": attn, "mlp": mlp}


def train_predictors(model: M.Model, traces, cfg: PredictorTrainConfig, rank: int | None = None, seed: int = 0,
                     out_path=None) -> tuple[dict, dict]:
    """run_train_predictors (sf/harness.py:320-371): per-layer training on the first 80% of the
    traces, held-out pattern agreement and MLP recall / precision on the rest."""
    dims = model.dims
    n_train = max(1, int(0.8 * len(traces)))
    train, held = traces[:n_train], traces[n_train:] or traces[:1]
    rank = rank or max(4, dims.d_model // 16)
    preds = {"attn": [], "mlp": []}
    attn_losses, mlp_losses = [], []
    for layer in range(dims.n_layers):
        ap = init_attn_predictor(dims.d_model, dims.n_heads, rank=rank, seed=seed + 100 + layer)
        attn_losses.append(train_attn_predictor([t[layer]["x_attn_ds"] for t in train], [t[layer]["raw_ds"] for t in train],
                                                ap, cfg, seed=seed + 200 + layer, device=model.device))
        preds["attn"].append(ap)
        mp = init_mlp_predictor(dims.d_model, dims.n_blk, seed=seed + 300 + layer)
        mlp_losses.append(train_mlp_predictor([t[layer]["x_mlp"] for t in train], [t[layer]["active_bits"] for t in train],
                                              dims.n_blk, mp, cfg, seed=seed + 400 + layer, device=model.device))
        preds["mlp"].append(mp)
    agree = total = 0
    recalls, precisions = [], []
    dev = model.device
    for t in held:
        for layer in range(dims.n_layers):
            rec = t[layer]
            xs = torch.as_tensor(np.asarray(rec["x_attn_ds"], np.float32), device=dev).to(torch.bfloat16)
            idx, _ = attn_pattern_idx(xs, 1, xs.shape[0], preds["attn"][layer], model.dpool, dims.n_b, cfg)
            grids = np.stack([upsample_mask(binarize_scores(r, cfg.attn_threshold_frac), dims.n_b) for r in rec["raw_ds"]])
            truth = EX.select_by_coverage(torch.as_tensor(grids.astype(np.float64), device=dev)[None], model.dpool,
                                          cfg.tau_pred)
            agree += int((idx[0] == truth[0]).sum())
            total += dims.n_heads
            s_hat = approx_mlp_scores(torch.as_tensor(np.asarray(rec["x_mlp"], np.float32), device=dev), preds["mlp"][layer])
            pred_mask = (s_hat > cfg.mlp_threshold).any(dim=0)
            truth_mask = bits_to_bool(torch.as_tensor(rec["active_bits"]).to(dev), dims.n_blk).any(dim=0)
            r, p = eval_recall_precision(pred_mask, truth_mask)
            recalls.append(r)
            precisions.append(p)
    if out_path is not None:
        save_predictors(out_path, preds)
    return preds, {
        "attn_final_loss": [round(x, 9) for x in attn_losses],
        "mlp_final_loss": [round(x, 9) for x in mlp_losses],
        "attn_pattern_agreement": round(agree / total, 9),
        "mlp_recall": round(float(np.mean(recalls)), 9),
        "mlp_precision": round(float(np.mean(precisions)), 9),
    }
