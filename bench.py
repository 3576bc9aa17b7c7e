#!/usr/bin/env python
"""Headline benchmark: OPT-1.3B LoRA fine-tune step (fwd + bwd + Adam) in
predicted mode on B200 — BASELINE.json metric "OPT-1.3B LoRA fwd+bwd ms/batch"
at configs[2] (batch 8, seq 512, bf16).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config cfg3]
    torchrun --nproc-per-node N bench.py --gpus N ...   (data parallel, NCCL)

`--gpus N > 1` without a torchrun environment re-launches this script under
torch.distributed.run with N ranks; it exits non-zero when fewer than N GPUs
are visible, or when WORLD_SIZE disagrees with --gpus.

Data parallel by batch with STRONG scaling: the global batch
G (the config's B) is split contiguously over the ranks (dp.shard_range), each
rank runs its shard, and the only collective is the flat trainable-gradient
all-reduce (NCCL) before the replicated Adam step.

Prints ONE JSON line (rank 0):
  value     device time per global batch, max over ranks: CUDA events around K
            CUDA-graph replays of the whole step, inputs resident;
  e2e       the same step through the public engine API (FinetuneEngine.replay)
            timed on the HOST clock: every step copies its token batch from pinned
            host memory and reads the loss back to the host (sf/harness.py:423-425);
  roofline  the dominant hot-path kernel (largest device time in one eager step,
            CUDA events around each launch on its stream) against MEASURED_PEAKS;
  kernels   the same for every timed hot-path kernel, with algorithmic units;
  cpu_baseline  the reference algorithm (oracle/ NumPy port) on the host cores.
Sparsity is injected through the predictor weights and the predictor kernels
run for real: MLP predictor columns zeroed for a fraction of neuron blocks, and
on a fraction of the heads Gram attention predictors (Wq_hat = Wk_hat) with the
residual stream's common mode projected out (calibrated layer by layer in one
predicted-mode forward), which the device predictor turns into block-diagonal
patterns. The achieved
sparsity is reported beside the number.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    # BASELINE.json configs[2]: OPT-1.3B (public OPT dims), LoRA r=8 on wq/wv/w1/w2, global batch 8, seq 512
    "cfg3": dict(d=2048, H=32, d_ff=8192, L=24, V=50272, B=8, s=512, blk=16, attn_blk=64, r=8, desc="OPT-1.3B"),
    # configs[3]: OPT-6.7B (d 4096, hd 128), seq 1024, global batch 16, LoRA / Adapter / BitFit
    "cfg4": dict(d=4096, H=32, d_ff=16384, L=32, V=50272, B=16, s=1024, blk=16, attn_blk=64, r=8, desc="OPT-6.7B"),
    # configs[4]: OPT-13B (d 5120, H 40, hd 128), seq 2048, global batch 8 (one sequence per GPU at 8 GPUs)
    "cfg5": dict(d=5120, H=40, d_ff=20480, L=40, V=50272, B=8, s=2048, blk=16, attn_blk=128, r=8, desc="OPT-13B"),
    # configs[0] shape (OPT-125M), batch 1 seq 256
    "cfg1": dict(d=768, H=12, d_ff=3072, L=12, V=50272, B=1, s=256, blk=16, attn_blk=16, r=8, desc="OPT-125M"),
}

# kernels of ours launched per C-ABI call (for gpu_launches)
KERNELS_PER_CALL = {
    "lx_gemm_bf16_tn": 1, "lx_linear": 1, "lx_linear_kn": 1, "lx_cross_entropy": 1, "lx_adam_step": 1, "lx_predict_mlp_mask": 2, "lx_mask_compact": 1,
    "lx_predict_attention_patterns": 2, "lx_neuron_fc1": 1, "lx_neuron_fc2": 1, "lx_neuron_fc2_dgrad": 1, "lx_neuron_fc1_dgrad": 1,
    "lx_rowproj": 2, "lx_rowproj_packed": 1, "lx_rowproj_packed_seg": 1, "lx_pack_params": 1, "lx_pack_active_rows": 1, "lx_pack_active_rows2": 1, "lx_lm_head_ce": 3, "lx_colgrad_group": 3,
    "lx_bsattn_fwd": 1, "lx_bsattn_bwd": 3, "lx_bsattn_fwd_tc": 1, "lx_bsattn_bwd_tc": 3, "lx_layernorm_fwd": 1,
    "lx_layernorm_bwd": 1, "lx_adapter_fwd": 1, "lx_adapter_bwd": 3,
}

# hot-path C-ABI calls timed by the roofline probe
PROBED = ("lx_neuron_fc1", "lx_neuron_fc2", "lx_neuron_fc2_dgrad", "lx_neuron_fc1_dgrad", "lx_bsattn_fwd_tc",
          "lx_bsattn_bwd_tc", "lx_predict_mlp_mask", "lx_predict_attention_patterns")


def load_peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm": d["hbm_gbs"], "bf16": d["bf16_tflops"], "bf16_sust": d.get("bf16_tflops_sustained", d["bf16_tflops"]),
                "src": "measured"}
    return {"hbm": 6650.0, "bf16": 1590.0, "bf16_sust": 1400.0, "src": "fallback"}


class ClockSampler:
    """nvidia-smi-equivalent sampling (NVML) of SM clock and throttle reasons during the timed region."""

    def __init__(self, index: int):
        self.index, self.samples, self.reasons, self._stop = index, [], set(), threading.Event()
        self.max_mhz = None

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        except Exception:  # pragma: no cover
            self._nv = None
        return self

    def _run(self):
        nv = self._nv
        names = {getattr(nv, k): k.replace("nvmlClocksThrottleReason", "").replace("nvmlClocksEventReason", "")
                 for k in dir(nv) if k.startswith(("nvmlClocksThrottleReason", "nvmlClocksEventReason")) and
                 isinstance(getattr(nv, k), int) and getattr(nv, k) not in (0,)}
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h) if hasattr(nv, "nvmlDeviceGetCurrentClocksEventReasons") \
                    else nv.nvmlDeviceGetCurrentClocksThrottleReasons(self._h)
                for bit, name in names.items():
                    if bit and (r & bit) == bit and bin(bit).count("1") == 1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.05)

    def __exit__(self, *a):
        self._stop.set()
        if self._nv is not None:
            self._t.join(timeout=1)

    def summary(self) -> dict:
        reasons = sorted(r for r in self.reasons if r not in ("GpuIdle", "ApplicationsClocksSetting"))
        return {"sm_mhz": float(statistics.median(self.samples)) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.samples)}


# ---------------------------------------------------------------------------- workload


class _CalibratingProvider:
    """One forward in which each layer's attention predictor is built from the LN1 output the layer
    actually receives (so from the predicted patterns / masks of all earlier layers): heads < n_local get
    a Gram predictor W_q = W_k = (I - U U^T) R, U the layer's k_shared dominant row directions (top right
    singular vectors of the LN1 output: the residual stream's common mode and the components that blocks of
    tokens share); the remaining heads independent random factors (N(0, 0.1^2), sf/predictor.py:194-206).
    Without the projection every token pair shares those directions and the Gram map is dense."""

    fused_downsample = False

    def __init__(self, inner, n_local: int, r_pred: int, g, device, k_shared: int = int(os.environ.get("LX_BENCH_KSHARED", "32"))):
        self.inner, self.n_local, self.r_pred, self.g, self.device = inner, n_local, r_pred, g, device
        self.k_shared = k_shared

    def attn_patterns(self, layer, h, x_small=None):
        import torch

        from paper_2510_15964_b200 import predictor as P

        d = h.shape[-1]
        H = self.inner.model.dims.n_heads
        # the shared directions of the layer's rows: the top singular vectors of the LN1 output (the mean
        # direction first); projecting them out of R leaves token-specific directions only
        _, _, vh = torch.linalg.svd(h.float().reshape(-1, d), full_matrices=False)
        U = vh[: self.k_shared].t().contiguous()  # [d, k]
        wq, wk = [], []
        for hh in range(H):
            w = torch.randn(d, self.r_pred, generator=self.g, device=self.device) * 0.1
            if hh < self.n_local:
                w = w - U @ (U.t() @ w)
                wq.append(w)
                wk.append(w)
            else:
                wq.append(w)
                wk.append(torch.randn(d, self.r_pred, generator=self.g, device=self.device) * 0.1)
        ap = P.AttnPredictorParams(wq, wk)
        ap.packed_t(self.device)  # device copy [2*H*r, d] bf16; drop the fp32 factors (shape-only meta tensors)
        ap.wq_hat = ap.wk_hat = [torch.empty(d, self.r_pred, device="meta") for _ in range(H)]
        self.inner.predictors["attn"][layer] = ap
        return self.inner.attn_patterns(layer, h)

    def mlp_mask(self, layer, h):
        return self.inner.mlp_mask(layer, h)


def build_workload(cfg: dict, device, seed: int, mlp_sparsity: float, local_frac: float, peft: str = "lora"):
    import torch

    from paper_2510_15964_b200 import harness as HN, model as M, predictor as P

    dims = M.ModelDims(cfg["d"], cfg["H"], cfg["d_ff"], cfg["s"], cfg["L"], cfg["V"], cfg["blk"], cfg["attn_blk"])
    model = M.build_model(dims, seed=seed, peft=peft, lora_rank=cfg["r"], device=device)
    g = torch.Generator(device=device).manual_seed(seed + 1)
    for ad in model.lora.values():  # LoRA-B off its zero init so every LoRA path carries signal
        ad.b.normal_(0.0, 0.02, generator=g)
    for ad in model.adapters.values():
        ad.w_up.normal_(0.0, 0.02, generator=g)
    d, H, n_blk = dims.d_model, dims.n_heads, dims.n_blk
    n_local = int(round(H * local_frac))
    if os.environ.get("LX_BENCH_IDENTITY_QK", "1") == "1":
        # pkg/demos/01_expose_sparsity.py:20-42: the local heads' q/k projections become scaled identities on the
        # head slice (3 I), so each token's score concentrates on itself and similar tokens
        hd = dims.head_dim
        eye = 3.0 * torch.eye(hd, device=device, dtype=torch.bfloat16)
        for lw in model.weights.layers:
            for off in (0, d):  # W_q | W_k column blocks of the fused [d, 3d] projection
                for h in range(n_local):
                    c0 = off + h * hd
                    lw.wqkv[:, c0 : c0 + hd] = 0
                    lw.wqkv[h * hd : (h + 1) * hd, c0 : c0 + hd] = eye
    state = M.make_peft_state(model)
    r_pred = max(4, d // 16)  # sf/harness.py:332 default
    mlp = []
    for layer in range(dims.n_layers):
        wa = torch.randn(d, n_blk, generator=g, device=device) * 0.1
        kill = torch.randperm(n_blk, generator=torch.Generator().manual_seed(seed * 131 + layer))[: int(round(mlp_sparsity * n_blk))]
        wa[:, kill.to(device)] = 0.0  # S_hat = 0 -> never > 0 -> block inactive (sparsity injection)
        mp = P.MlpPredictorParams(wa)
        mp.packed_t(device)
        mp.wa_hat = None
        mlp.append(mp)
    provider = HN.PredictedProvider(model, {"attn": [None] * dims.n_layers, "mlp": mlp}, P.PredictorTrainConfig())
    # calibration forward on one synthetic sequence builds every layer's attention predictor in place
    tok = torch.randint(0, dims.vocab, (1, dims.seq_len), generator=torch.Generator().manual_seed(seed + 4242)).to(device)
    with torch.no_grad():
        M.model_forward(model, tok, _CalibratingProvider(provider, n_local, r_pred, g, device))
    provider.reset_timing()
    return model, state, provider


def count_launches(fn) -> int:
    from paper_2510_15964_b200 import _abi

    n = [0]
    orig = _abi.call

    def counting(name, *args):
        n[0] += KERNELS_PER_CALL.get(name, 0)
        return orig(name, *args)

    _abi.call = counting
    try:
        fn()
    finally:
        _abi.call = orig
    return n[0]


def achieved_sparsity(masks, model) -> dict:
    from paper_2510_15964_b200.model import dp_nnz

    dims = model.dims
    nnz_of = {i: dp_nnz(model.dpool, i) for i in range(len(model.dpool.ids))}
    nm_density, at_density = [], []
    for lm in masks:
        nm_density.append(float(lm.neuron_mask.counts.float().mean()) / dims.n_blk)
        idx = lm.head_patterns.flatten().tolist()
        at_density.append(float(np.mean([nnz_of[i] for i in idx])) / dims.n_b ** 2)
    return {"mlp_block_sparsity": round(1 - float(np.mean(nm_density)), 4),
            "attn_block_sparsity": round(1 - float(np.mean(at_density)), 4)}


def _max_over_ranks(x: float, dist, device) -> float:
    if dist is None:
        return x
    import torch

    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def time_graph(engine, K: int, dist, device) -> float:
    import torch

    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st.record()
    for _ in range(K):
        engine.replay()
    en.record()
    torch.cuda.synchronize()
    return _max_over_ranks(st.elapsed_time(en) / K, dist, device)


class StateSnapshot:
    """Trainable parameters, Adam moments and step count; rank-0-only probe steps run between
    snapshot and restore so every rank ends with the state the timed steps left."""

    def __init__(self, state):
        self.state = state
        self.saved = (state.flat.clone(), state.m.clone(), state.v.clone(), state.step)

    def restore(self):
        f, m, v, step = self.saved
        self.state.flat.copy_(f)
        self.state.m.copy_(m)
        self.state.v.copy_(v)
        self.state.step = step


def kernel_probe(model, engine, tok_dev, peaks: dict, config: str) -> tuple[dict, list]:
    """Time every probed hot-path call of one eager training step (CUDA events around each launch on its
    stream; the GPU is held ~1 s first so the whole step is queued and the events bracket GPU execution
    only) and credit algorithmic units per launch:
      fc GEMMs   2 * s * d * sum_b counts_b * blk FLOPs
      attention  fwd 4 * sum_(b,h) nnz * attn_blk^2 * hd, bwd 8 * (...) FLOPs (reference MAC convention)
      K1 mask    HBM bytes: MLP = M*d*2 (h2) + n_blk*d*4 (fp32 W_a) + outputs; attention = B*m*d*2 + 2*H*r*d*4.
    Returns (dominant kernel's roofline object, per-kernel list)."""
    import torch

    from paper_2510_15964_b200 import _abi
    from paper_2510_15964_b200.model import dp_nnz
    from paper_2510_15964_b200.predictor import downsample_indices

    dims = model.dims
    _abi.PROBE = {n: [] for n in PROBED}
    try:
        torch.cuda._sleep(2_000_000_000)
        engine.step(tok_dev)
        torch.cuda.synchronize()
        rec = _abi.PROBE
    finally:
        _abi.PROBE = None
    masks = engine.last_masks
    L, s, d, hd, blk, ab = dims.n_layers, dims.seq_len, dims.d_model, dims.head_dim, dims.blk_size, dims.attn_blk
    B = int(masks[0].neuron_mask.counts.numel())
    nnz_of = {i: dp_nnz(model.dpool, i) for i in range(len(model.dpool.ids))}
    fc_fl = [2.0 * s * d * float(lm.neuron_mask.counts.sum()) * blk for lm in masks]
    att_nnz = []
    for lm in masks:
        hp = lm.head_patterns
        n = sum(nnz_of[i] for i in hp.flatten().tolist())
        att_nnz.append(n * (B if hp.shape[0] == 1 else 1))
    # executed tensor work of the attention kernels: MMAs per gathered 128-tile entry (fwd: S, PV; bwd: dK/dV
    # kernel S, dV, dP, dK over the CSC entries + dQ kernel S, dP, dQ over the CSR entries), 2 * 128 * 128 * hd each
    tab = model.dpool.tables.cpu().numpy() if model.dpool.tables is not None else None
    ent_csr, ent_csc = [], []
    for lm in masks:
        hp = lm.head_patterns.flatten().tolist()
        mult = B if lm.head_patterns.shape[0] == 1 else 1
        if tab is None:
            ent_csr.append(0)
            ent_csc.append(0)
            continue
        nt, per = int(tab[0]), int(tab[6])
        ent_csr.append(mult * sum(int(tab[8 + i * per + nt]) for i in hp))
        ent_csc.append(mult * sum(int(tab[8 + i * per + 2 * nt + 1]) for i in hp))
    mma = 2.0 * 128 * 128 * hd
    executed = {"lx_bsattn_fwd_tc": [2 * mma * e for e in ent_csr],
                "lx_bsattn_bwd_tc": [mma * (4 * c + 3 * r) for r, c in zip(ent_csr[::-1], ent_csc[::-1])]}
    m = len(downsample_indices(s))
    r_pred = max(4, d // 16)
    units = {
        "lx_neuron_fc1": ("tensor", fc_fl), "lx_neuron_fc2": ("tensor", fc_fl),
        "lx_neuron_fc2_dgrad": ("tensor", fc_fl[::-1]), "lx_neuron_fc1_dgrad": ("tensor", fc_fl[::-1]),
        "lx_bsattn_fwd_tc": ("tensor", [4.0 * n * ab * ab * hd for n in att_nnz]),
        "lx_bsattn_bwd_tc": ("tensor", [8.0 * n * ab * ab * hd for n in att_nnz[::-1]]),
        "lx_predict_mlp_mask": ("hbm", [float(B * s * d * 2 + dims.n_blk * d * 4 + 4 * B * (2 * dims.n_blk + 1))] * L),
        # the predictor weights are float32 (sf/predictor.py): 4 B each, streamed as a bf16 hi/lo pair
        "lx_predict_attention_patterns": ("hbm", [float(B * m * d * 2 + 2 * dims.n_heads * r_pred * d * 4 + 4 * B * dims.n_heads)] * L),
    }
    traffic_db = {}
    prof = ROOT / "profiles" / "r02_ncu_traffic.json"
    if prof.exists():
        traffic_db = json.loads(prof.read_text()).get(config, {})
    out = []
    for name, evs in rec.items():
        if not evs:
            continue
        bound, work = units[name]
        ms = [a.elapsed_time(b) for a, b in evs]
        n = min(len(ms), len(work))
        ms_avg = statistics.mean(ms[:n])
        w_avg = statistics.mean(work[:n])
        if bound == "tensor":
            ach, peak, unit = w_avg / (ms_avg * 1e-3) / 1e12, peaks["bf16_sust"], "TFLOP/s"
        else:
            ach, peak, unit = w_avg / (ms_avg * 1e-3) / 1e9, peaks["hbm"], "GB/s"
        out.append({"kernel": name, "bound": bound, "achieved": round(ach, 1), "peak": peak, "unit": unit,
                    "frac": round(ach / peak, 4), "traffic": traffic_db.get(name), "ms_per_launch": round(ms_avg, 4),
                    "launches": len(ms), "total_ms": round(sum(ms), 3),
                    ("flops_per_launch" if bound == "tensor" else "bytes_per_launch"): w_avg})
        if name in executed and executed[name][:n]:
            # context, not the roofline: the MMA work the 128-tile kernels issue (active cells padded to 128 x 128
            # gathered tiles, the flash recompute included) against the same peak
            ex = statistics.mean(executed[name][:n])
            out[-1]["executed_flops_per_launch"] = ex
            out[-1]["executed_frac"] = round(ex / (ms_avg * 1e-3) / 1e12 / peak, 4)
    out.sort(key=lambda k: -k["total_ms"])
    dom = dict(out[0])
    dom["peak_src"] = (f"{peaks['src']} " + ("sustained bf16 (kernel timed inside the step)" if dom["bound"] == "tensor"
                                             else "HBM copy bandwidth"))
    dom["timing"] = "CUDA events around each launch of one eager step (all layers) on the launching stream, mean"
    return dom, out


def k1_summary(kernels) -> dict | None:
    """K1 (predictor scoring + exposer aggregation -> masks / patterns) per layer: both calls' time and algorithmic
    HBM bytes (fp32 predictor weights, bf16 activations, index outputs) -> achieved GB/s against the HBM peak."""
    k = [x for x in kernels or [] if x["kernel"].startswith("lx_predict")]
    if not k:
        return None
    us = sum(x["ms_per_launch"] for x in k) * 1e3
    by = sum(x["bytes_per_launch"] for x in k)
    tr = [x.get("traffic") for x in k]
    return {"calls": [x["kernel"] for x in k], "us_per_layer": round(us, 2), "bytes_per_layer": by,
            "achieved": round(by / (us * 1e-6) / 1e9, 1), "unit": "GB/s", "peak": k[0]["peak"],
            "frac": round(by / (us * 1e-6) / 1e9 / k[0]["peak"], 4),
            "traffic": sum(tr) if all(t is not None for t in tr) else None}


def run_ours(args, cfg, rank, world, dist):
    import torch

    from paper_2510_15964_b200 import harness as HN
    from paper_2510_15964_b200.dense_baseline import DenseLoraStep
    from paper_2510_15964_b200.dp import BucketedGradSync, shard_range
    from paper_2510_15964_b200.engine import FinetuneEngine

    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    peaks = load_peaks()
    G = cfg["B"]
    b0, b1 = shard_range(G, rank, world)
    B = b1 - b0
    model, state, provider = build_workload(cfg, dev, seed=args.seed, mlp_sparsity=args.mlp_sparsity,
                                            local_frac=args.local_frac, peft=args.peft)
    # the only collective: the flat trainable-gradient all-reduce, bucketed per layer group and overlapped with the
    # backward on a communication stream (NCCL, captured in the step's CUDA graph)
    sync = BucketedGradSync(dist, G, rank, world) if dist is not None else None
    eng = FinetuneEngine(model, state, provider, lr=1e-4, grad_sync=sync)
    s, V = cfg["s"], cfg["V"]
    gen = torch.Generator().manual_seed(args.seed + 2)  # synthetic uniform tokens (sf/harness.py:391 seed + 2)
    batches = [torch.randint(0, V, (G, s + 1), generator=gen)[b0:b1].contiguous() for _ in range(max(args.steps, 1))]
    tok_dev = batches[0].to(dev)
    for _ in range(max(args.warmup - 1, 1)):
        eng.step(tok_dev)
    per_step = count_launches(lambda: eng.step(tok_dev))
    torch.cuda.synchronize()
    eng.capture(tok_dev, warmup=1)
    eng.replay()
    torch.cuda.synchronize()
    with ClockSampler(dev.index) as clk:
        ms = time_graph(eng, args.steps, dist, dev)
    sparsity = achieved_sparsity(eng.last_masks, model)
    # e2e through the public API on the host clock: pinned host batch -> device, step, loss -> host, every step
    pinned = [b.pin_memory() for b in batches]
    loss_host = torch.empty((), dtype=torch.float32).pin_memory()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    losses = []
    for k in range(args.steps):
        loss = eng.replay(pinned[k % len(pinned)])
        loss_host.copy_(loss)  # blocking device->host read: the host has the loss before the next step starts
        losses.append(float(loss_host))
    e2e_ms = (time.perf_counter() - t0) * 1e3 / args.steps
    e2e_ms = _max_over_ranks(e2e_ms, dist, dev)
    extra = {}
    roof, kernels = None, None
    if rank == 0:
        snap = StateSnapshot(state)  # rank-0-only probes below must not leave rank 0's state diverged
        eng.graph = eng.static_loss = None  # the step graph's memory pool back before the eager probe / dense steps
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        sync_saved, eng.grad_sync = eng.grad_sync, None  # rank-0-only probe step: no collective
        roof, kernels = kernel_probe(model, eng, tok_dev, peaks, args.config)
        eng.grad_sync = sync_saved
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        if not args.skip_dense:
            # dense reference points on the same box: (a) same engine, every head/block dense; (b) torch cuBLAS/SDPA
            dprov = HN.DenseProvider(model)
            deng = FinetuneEngine(model, state, dprov, lr=1e-4)
            deng.step(tok_dev)
            deng.capture(tok_dev, warmup=1)
            extra["dense_same_kernels_ms"] = round(time_graph(deng, max(3, args.steps // 2), None, dev), 3)
            extra["speedup_vs_dense_same_kernels"] = round(extra["dense_same_kernels_ms"] / ms, 3)
            del deng, dprov
            torch.cuda.synchronize()
            torch.cuda.empty_cache()
            if args.peft == "lora":
                try:
                    tstep = DenseLoraStep(model, lr=1e-4)
                    tstep.capture(tok_dev)
                    torch.cuda.synchronize()
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    n = max(3, args.steps // 2)
                    a.record()
                    for _ in range(n):
                        tstep.replay()
                    b.record()
                    torch.cuda.synchronize()
                    extra["dense_torch_ms"] = round(a.elapsed_time(b) / n, 3)
                    extra["speedup_vs_dense_torch"] = round(extra["dense_torch_ms"] / ms, 3)
                    extra["dense_torch"] = ("CUDA-graphed torch bf16 step: cuBLAS GEMMs, SDPA, chunked fused LM-head CE, "
                                            "fused capturable Adam (paper_2510_15964_b200/dense_baseline.py), same B")
                    del tstep
                except Exception as e:  # pragma: no cover
                    extra["dense_torch_error"] = repr(e)[:200]
        snap.restore()
    cpu = None
    if rank == 0 and world == 1 and not args.skip_cpu:
        cpu = cpu_baseline(cfg, args)
    frozen_gb = sum(t.numel() * t.element_size() for lw in model.weights.layers
                    for t in (lw.wqkv, lw.wo, lw.mlp.w1_t, lw.mlp.w2)) / 1e9
    tokens_per_step = G * s
    line = {
        "metric": f"{cfg['desc']} {args.peft.upper() if args.peft != 'lora' else 'LoRA'} fwd+bwd ms/batch",
        "value": round(ms, 3), "unit": "ms/batch", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic (uniform tokens, random-init weights)",
        "config": {"workload": (f"{args.config}: {cfg['desc']} {args.peft} fine-tune step (predict+fwd+bwd+Adam), predicted "
                                f"mode, global batch {G} split over {world} GPU(s)"),
                   "model": cfg["desc"], "peft": args.peft, "global_batch": G, "per_rank_batch": B, "seq_len": s,
                   "parallelism": f"dp{world}", "d_model": cfg["d"], "n_layers": cfg["L"], "d_ff": cfg["d_ff"], "vocab": V,
                   "blk_size": cfg["blk"], "attn_blk": cfg["attn_blk"], "lora_rank": cfg["r"], "mask_scope": "per sequence",
                   **sparsity,
                   "injected": {"mlp_zeroed_predictor_blocks": args.mlp_sparsity,
                                "calibrated_gram_attention_heads": args.local_frac},
                   "l2": f"inputs larger than L2: {frozen_gb:.1f} GB of frozen weights stream from HBM every step (no flush needed)",
                   "timing": "CUDA events around K CUDA-graph replays (max over ranks); the bucketed gradient all-reduce "
                             "inside the graph, Adam (fp64 moments) after it, both inside the timed region"},
        "tokens_per_s": round(tokens_per_step / (ms * 1e-3), 1),
        "e2e": {"value": round(e2e_ms, 3), "unit": "ms/batch", "h2d_bytes_per_step": int(G * (s + 1) * 8),
                "d2h_bytes_per_step": 4 * world,
                "api": "FinetuneEngine.replay(pinned host batch) + blocking loss read to the host every step; host "
                       "perf_counter, max over ranks",
                "tokens_per_s": round(tokens_per_step / (e2e_ms * 1e-3), 1)},
        "gpu_launches": int(per_step * args.steps), "gpu_launches_per_step": int(per_step),
        "final_loss": round(losses[-1], 5),
        "clocks": clk.summary(),
        "roofline": roof,
        "k1": k1_summary(kernels),
        "kernels": kernels,
        "cpu_baseline": cpu,
        **extra,
    }
    return line


# ---------------------------------------------------------------------------- CPU reference (oracle port)


def _blas_threads() -> int:
    try:
        from threadpoolctl import threadpool_info

        return max((i.get("num_threads", 1) for i in threadpool_info()), default=1)
    except Exception:  # pragma: no cover
        return os.cpu_count() or 1


def _oracle_setup(cfg: dict, args, n_layers: int, seed: int):
    from oracle import sf_oracle as O

    d, H, f, s, V = cfg["d"], cfg["H"], cfg["d_ff"], cfg["s"], cfg["V"]
    dims = O.Dims(d, H, f, s, n_layers, V, cfg["blk"], cfg["attn_blk"])
    om = O.build_model(dims, seed=seed, peft="lora", lora_rank=cfg["r"])
    rng = O.make_rng(seed + 1)
    n_blk, r_pred = dims.n_blk, max(4, d // 16)
    attn, mlp = [], []
    n_local = int(round(H * args.local_frac))
    for _ in range(n_layers):
        wq = [O.randn(rng, (d, r_pred), 0.1) for _ in range(H)]
        wk = [wq[h] if h < n_local else O.randn(rng, (d, r_pred), 0.1) for h in range(H)]
        attn.append(O.AttnPredictorParams(wq, wk))
        wa = O.randn(rng, (d, n_blk), 0.1)
        wa[:, rng.permutation(n_blk)[: int(round(args.mlp_sparsity * n_blk))]] = 0.0
        mlp.append(O.MlpPredictorParams(wa))
    return O, om, O.PredictedProvider(om, attn, mlp, O.PredictorConfig()), rng


def cpu_sample(cfg: dict, args, n_layers_sample: int = 2):
    """One bounded sample of the reference step (sf/harness.py:401-417 on the oracle, predicted mode):
    one sequence through `n_layers_sample` layers + LM head + loss + backward + Adam. Returns a callable
    that runs the sample and returns the extrapolation to the full batch (G sequences, L layers) in ms."""
    O, om, prov, rng = _oracle_setup(cfg, args, n_layers_sample, args.seed)
    s, V = cfg["s"], cfg["V"]
    seq = rng.integers(0, V, size=s + 1)
    tok, tgt = seq[:-1], seq[1:]
    params = O.trainable_params(om)

    def one() -> dict:
        t = {}
        t0 = time.perf_counter()
        h = om.emb[tok]
        caches = []
        for i in range(n_layers_sample):
            h, c = O.block_forward(h, om, i, prov)
            caches.append(c)
        t["layers_fwd"] = time.perf_counter() - t0
        t1 = time.perf_counter()
        hf, cf = O.layernorm_forward(h, om.lnf_g, om.lnf_b)
        logits = hf @ om.emb.T
        O.loss_forward(logits, tgt)
        dl = O.loss_backward(logits, tgt)
        dh = O.layernorm_backward(dl @ om.emb, cf)
        t["head"] = time.perf_counter() - t1
        t2 = time.perf_counter()
        grads = {}
        for i in reversed(range(n_layers_sample)):
            dh = O.block_backward(dh, om, i, caches[i], grads)
        t["layers_bwd"] = time.perf_counter() - t2
        t3 = time.perf_counter()
        O.optimizer_step(params, {}, {}, 0, {k: grads.get(k, np.zeros_like(v)) for k, v in params.items()}, 1e-4)
        t["adam"] = time.perf_counter() - t3
        per_layer = (t["layers_fwd"] + t["layers_bwd"]) / n_layers_sample
        t["extrapolated_ms"] = (cfg["B"] * (per_layer * cfg["L"] + t["head"]) + t["adam"] * cfg["L"] / n_layers_sample) * 1e3
        t["per_layer_ms"] = per_layer * 1e3
        return t

    return one


def cfg1_measured(args) -> dict:
    """The reference's own CPU-runnable config (BASELINE configs[0]) timed for real: the full OPT-125M-shaped
    predicted-mode LoRA step, B=1, s=256, 12 layers (sf/harness.py:401-417), 1 warm-up + median of 3."""
    c1 = CONFIGS["cfg1"]
    O, om, prov, rng = _oracle_setup(c1, args, c1["L"], args.seed)
    seq = rng.integers(0, c1["V"], size=(1, c1["s"] + 1))
    params = O.trainable_params(om)
    mom, vel, step = {}, {}, 0
    ts = []
    for k in range(4):
        t0 = time.perf_counter()
        _, _, step = O.finetune_step(om, seq, prov, params, mom, vel, step, 1e-4)
        ts.append(time.perf_counter() - t0)
    return {"value": round(statistics.median(ts[1:]) * 1e3, 1), "unit": "ms/batch", "config": "cfg1 (OPT-125M shape, B=1, s=256, L=12)",
            "runs": "1 warm-up + median of 3", "extrapolated": False}


def cpu_baseline(cfg: dict, args) -> dict:
    one = cpu_sample(cfg, args)
    one()  # warm-up
    runs = [one() for _ in range(2)]
    med = statistics.median(r["extrapolated_ms"] for r in runs)
    per_layer = statistics.median(r["per_layer_ms"] for r in runs)
    return {"value": round(med, 1), "unit": "ms/batch", "cores": int(_blas_threads()), "kind": "port",
            "sample": (f"1 sequence x 2 of {cfg['L']} layers + LM head + Adam on the oracle (NumPy restatement of "
                       f"sf/harness.py:401-417, predicted mode, same injected sparsity), extrapolated x{cfg['B']} sequences "
                       f"x{cfg['L']}/2 layers; measured per-layer {per_layer:.0f} ms"),
            "extrapolated": True, "host_cpu_count": os.cpu_count(),
            "cfg1_measured": cfg1_measured(args) if not args.skip_cfg1 else None}


def run_reference(args, cfg, rank) -> dict | None:
    """The reference arm: the reference algorithm (oracle port of sf/, pure NumPy) on the host cores, rank 0 only.
    Each step is one bounded sample (1 sequence x 2 layers + head + Adam) extrapolated to ms per global batch."""
    if rank != 0:
        return None
    one = cpu_sample(cfg, args)
    t_start = time.perf_counter()
    for _ in range(args.warmup):
        one()
    vals = [one()["extrapolated_ms"] for _ in range(args.steps)]
    wall = time.perf_counter() - t_start
    v = statistics.median(vals)
    cores = int(_blas_threads())
    cpu = {"value": round(v, 1), "unit": "ms/batch", "cores": cores, "kind": "port", "extrapolated": True,
           "sample": (f"each step: 1 sequence x 2 of {cfg['L']} layers + LM head + Adam of the oracle (NumPy restatement "
                      f"of sf/harness.py:401-417), extrapolated x{cfg['B']} sequences x{cfg['L']}/2 layers; "
                      f"{args.warmup + args.steps} samples ran in {wall:.1f} s"),
           "host_cpu_count": os.cpu_count(),
           "cfg1_measured": cfg1_measured(args) if not args.skip_cfg1 else None}
    return {"impl": "reference", "metric": f"{cfg['desc']} LoRA fwd+bwd ms/batch", "value": round(v, 1), "unit": "ms/batch",
            "n_gpus": int(os.environ.get("WORLD_SIZE", 1)), "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(v, 1), "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "config": {"workload": f"{args.config} (as ours), reference algorithm on host cores, "
                                                        "bounded samples extrapolated", "model": cfg["desc"],
                                            "global_batch": cfg["B"], "seq_len": cfg["s"], "parallelism": "host"},
            "cpu_baseline": cpu, "e2e": {"value": round(v, 1), "unit": "ms/batch", "h2d_bytes_per_step": 0,
                                         "d2h_bytes_per_step": 0},
            "wall_s": round(wall, 1)}


def _relaunch(args) -> int:
    """--gpus N > 1 outside torchrun: start N ranks under torch.distributed.run (127.0.0.1 rendezvous)."""
    import socket

    import torch

    n_vis = torch.cuda.device_count()
    if n_vis < args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} requested but only {n_vis} GPU(s) visible"}), flush=True)
        return 2
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}", "--master-addr",
           "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg3", choices=sorted(CONFIGS))
    ap.add_argument("--peft", default="lora", choices=["lora", "adapter", "bitfit"])
    ap.add_argument("--mlp-sparsity", type=float, default=0.85)
    ap.add_argument("--local-frac", type=float, default=0.75)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--global-batch", type=int, default=0, help="global batch (default: the config's B)")
    ap.add_argument("--skip-dense", action="store_true")
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--skip-cfg1", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    cfg = dict(CONFIGS[args.config])
    if args.global_batch:
        cfg["B"] = args.global_batch
    env_world = os.environ.get("WORLD_SIZE")
    world = int(env_world or 1)
    rank = int(os.environ.get("RANK", 0))
    if args.impl == "reference":
        line = run_reference(args, cfg, rank)
        if line is not None:
            print(json.dumps(line), flush=True)
        return 0
    if env_world is None and args.gpus > 1:
        return _relaunch(args)
    if world != args.gpus:
        print(json.dumps({"error": f"WORLD_SIZE={world} but --gpus {args.gpus}"}), flush=True)
        return 2
    import torch

    if torch.cuda.device_count() < 1 or (world > 1 and torch.cuda.device_count() < world):
        print(json.dumps({"error": f"{world} rank(s) need {world} visible GPU(s); found {torch.cuda.device_count()}"}),
              flush=True)
        return 2
    dist = None
    if world > 1:
        import torch.distributed as tdist

        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
        tdist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0))))
        dist = tdist
    line = run_ours(args, cfg, rank, world, dist)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
