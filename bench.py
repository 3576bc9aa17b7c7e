#!/usr/bin/env python
"""Headline benchmark: OPT-1.3B LoRA fine-tune step (fwd + bwd + Adam) in
predicted mode on B200 — BASELINE.json metric "OPT-1.3B LoRA fwd+bwd ms/batch"
at configs[2] (batch 8, seq 512, bf16).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...   (data parallel, NCCL)

Prints ONE JSON line (rank 0). `value` = device-timed ms per step of the whole
job (max over ranks; CUDA events around K CUDA-graph replays of the full step,
inputs resident), `e2e` = the same step through the public engine API with the
batch copied host->device and the loss device->host every step. Sparsity is
injected through the predictor weights (zeroed MLP scoring columns; Gram-form
attention predictors for local heads) and the predictor kernels run for real;
the achieved sparsity is reported beside every number. `cpu_baseline` and
`--impl reference` time the reference algorithm (oracle/ NumPy port) on the
host cores on a bounded sample and extrapolate (see `sample`).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    # BASELINE.json configs[2]: OPT-1.3B (public OPT dims), LoRA r=8 on wq/wv/w1/w2, batch 8, seq 512
    "cfg3": dict(d=2048, H=32, d_ff=8192, L=24, V=50272, B=8, s=512, blk=16, attn_blk=64, r=8, desc="OPT-1.3B"),
    # BASELINE.json configs[3]: OPT-6.7B (d 4096, hd 128), LoRA seq 1024; global batch 16 split over the GPUs
    # (B below is per rank at 8 GPUs; `--batch` overrides)
    "cfg4": dict(d=4096, H=32, d_ff=16384, L=32, V=50272, B=2, s=1024, blk=16, attn_blk=64, r=8, desc="OPT-6.7B"),
    # configs[0] shape (OPT-125M), batch 1 seq 256 — quick checks
    "cfg1": dict(d=768, H=12, d_ff=3072, L=12, V=50272, B=1, s=256, blk=16, attn_blk=64, r=8, desc="OPT-125M"),
}

# kernels of ours launched per C-ABI call (for gpu_launches)
KERNELS_PER_CALL = {
    "lx_gemm_bf16_tn": 1, "lx_linear": 1, "lx_cross_entropy": 1, "lx_adam_step": 1, "lx_predict_mlp_mask": 2, "lx_mask_compact": 1, "lx_predict_attention_patterns": 2,
    "lx_neuron_fc1": 1, "lx_neuron_fc2": 1, "lx_neuron_fc2_dgrad": 1, "lx_neuron_fc1_dgrad": 1, "lx_rowproj": 2, "lx_rowproj_packed": 1, "lx_pack_params": 1, "lx_pack_active_rows": 1,
    "lx_colgrad_group": 3, "lx_bsattn_fwd": 1, "lx_bsattn_bwd": 3, "lx_bsattn_fwd_tc": 1, "lx_bsattn_bwd_tc": 3, "lx_layernorm_fwd": 1, "lx_layernorm_bwd": 1,
}


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
            time.sleep(0.1)

    def __exit__(self, *a):
        self._stop.set()
        if self._nv is not None:
            self._t.join(timeout=1)

    def summary(self) -> dict:
        reasons = sorted(r for r in self.reasons if r not in ("GpuIdle", "ApplicationsClocksSetting"))
        return {"sm_mhz": float(statistics.median(self.samples)) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.samples)}


# ---------------------------------------------------------------------------- our arm


def build_workload(cfg: dict, device, seed: int, mlp_sparsity: float, local_frac: float):
    import torch

    from paper_2510_15964_b200 import harness as HN, model as M, predictor as P

    dims = M.ModelDims(cfg["d"], cfg["H"], cfg["d_ff"], cfg["s"], cfg["L"], cfg["V"], cfg["blk"], cfg["attn_blk"])
    model = M.build_model(dims, seed=seed, peft="lora", lora_rank=cfg["r"], device=device)
    g = torch.Generator(device=device).manual_seed(seed + 1)
    for ad in model.lora.values():  # LoRA-B off its zero init so every LoRA path carries signal
        ad.b.normal_(0.0, 0.02, generator=g)
    state = M.make_peft_state(model)
    d, H, n_blk = dims.d_model, dims.n_heads, dims.n_blk
    r_pred = max(4, d // 16)  # sf/harness.py:332 default
    attn, mlp = [], []
    n_local = int(round(H * local_frac))
    for layer in range(dims.n_layers):
        wq = [torch.randn(d, r_pred, generator=g, device=device) * 0.1 for _ in range(H)]
        wk = [wq[h] if h < n_local else torch.randn(d, r_pred, generator=g, device=device) * 0.1 for h in range(H)]
        ap = P.AttnPredictorParams(wq, wk)
        ap.packed_t(device)  # device copy [2*H*r, d] bf16; drop the fp32 factors (shape-only meta tensors)
        ap.wq_hat = ap.wk_hat = [torch.empty(d, r_pred, device="meta") for _ in range(H)]
        attn.append(ap)
        wa = torch.randn(d, n_blk, generator=g, device=device) * 0.1
        kill = torch.randperm(n_blk, generator=torch.Generator().manual_seed(seed * 131 + layer))[: int(round(mlp_sparsity * n_blk))]
        wa[:, kill.to(device)] = 0.0  # S_hat = 0 -> never > 0 -> block inactive (sparsity injection)
        mp = P.MlpPredictorParams(wa)
        mp.packed_t(device)
        mp.wa_hat = None
        mlp.append(mp)
    provider = HN.PredictedProvider(model, {"attn": attn, "mlp": mlp}, P.PredictorTrainConfig())
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


def achieved_sparsity(engine, model) -> dict:
    import torch

    dims = model.dims
    nm_density, at_density = [], []
    from paper_2510_15964_b200.model import dp_nnz

    nnz_of = {i: dp_nnz(model.dpool, i) for i in range(len(model.dpool.ids))}
    for lm in engine.last_masks:
        nm_density.append(float(lm.neuron_mask.counts.float().mean()) / dims.n_blk)
        idx = lm.head_patterns.flatten().tolist()
        at_density.append(float(np.mean([nnz_of[i] for i in idx])) / dims.n_b ** 2)
    return {"mlp_block_sparsity": round(1 - float(np.mean(nm_density)), 4),
            "attn_block_sparsity": round(1 - float(np.mean(at_density)), 4)}


def time_graph(engine, K: int, dist) -> float:
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
    ms = st.elapsed_time(en) / K
    if dist is not None:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    return ms


def fc1_roofline(model, engine, tok_dev, peaks: dict, config: str = "cfg3") -> dict:
    """Dominant sparse kernel: the fc1 packed-row GEMM (bias + LoRA + ReLU fused), timed live inside one
    eager training step with CUDA events around each of its L launches on the launching stream (so the
    L2 state is the step's own); algorithmic FLOPs per launch = 2 * s * d * sum_b(counts_b * blk)."""
    import torch

    from paper_2510_15964_b200 import neuron_ops as N

    N.FC1_EVENTS = []
    hook, engine.grad_hook = engine.grad_hook, None  # rank-0-only probe step: no collective
    try:
        # hold the GPU ~1 s so the whole eager step is queued before it runs: the events then bracket
        # GPU execution only (no host-enqueue gaps between an event and its kernel)
        torch.cuda._sleep(2_000_000_000)
        engine.step(tok_dev)
        torch.cuda.synchronize()
        recs = N.FC1_EVENTS
    finally:
        N.FC1_EVENTS = None
        engine.grad_hook = hook
    ms = [a.elapsed_time(b) for a, b, *_ in recs]
    flops = [2.0 * s * d * float(c.sum()) * blk for _, _, c, s, d, blk in recs]
    ms_avg, fl_avg = statistics.mean(ms), statistics.mean(flops)
    ach = fl_avg / (ms_avg * 1e-3) / 1e12
    traffic = None
    prof = ROOT / "profiles" / "r01_fc1_ncu.json"
    if prof.exists():  # ncu DRAM bytes of one fc1 launch, valid for the config it was captured on
        pj = json.loads(prof.read_text())
        if pj.get("config", "cfg3") == config:
            traffic = pj.get("dram_bytes_per_launch")
    return {"kernel": "gemm_sm100_kernel<kPackedN,kEpiFc1> (neuron_matmul_fwd1+b1+LoRA+ReLU over packed active W1 rows)",
            "bound": "tensor", "achieved": round(ach, 1), "peak": peaks["bf16_sust"], "unit": "TFLOP/s",
            "frac": round(ach / peaks["bf16_sust"], 4), "traffic": traffic,
            "peak_src": f"{peaks['src']} sustained bf16 (kernel timed inside the step)",
            "ms_per_launch": round(ms_avg, 4), "flops_per_launch": fl_avg, "launches_timed": len(recs),
            "timing": "CUDA events around each fc1 launch of one eager step (all layers), mean"}


def run_ours(args, cfg, rank, world, dist):
    import torch

    from paper_2510_15964_b200 import harness as HN
    from paper_2510_15964_b200.dense_baseline import DenseLoraStep
    from paper_2510_15964_b200.engine import FinetuneEngine

    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)) % max(torch.cuda.device_count(), 1))
    torch.cuda.set_device(dev)
    peaks = load_peaks()
    model, state, provider = build_workload(cfg, dev, seed=args.seed, mlp_sparsity=args.mlp_sparsity,
                                            local_frac=args.local_frac)
    from paper_2510_15964_b200.dp import make_grad_hook

    # weak scaling: each rank runs its own B-sequence shard of a global batch of B*world
    hook = make_grad_hook(dist, cfg["B"] * world, rank, world) if dist is not None else None
    eng = FinetuneEngine(model, state, provider, lr=1e-4, grad_hook=hook)
    B, s, V = cfg["B"], cfg["s"], cfg["V"]
    gen = torch.Generator().manual_seed(args.seed + 2 + rank)  # synthetic uniform tokens, per-rank shard
    batches = [torch.randint(0, V, (B, s + 1), generator=gen) for _ in range(max(args.steps, 1))]
    tok_dev = batches[0].to(dev)
    # warm-up (eager; first calls set kernel attributes), then capture the step
    for _ in range(max(args.warmup - 1, 1)):
        eng.step(tok_dev)
    per_step = count_launches(lambda: eng.step(tok_dev))
    torch.cuda.synchronize()
    eng.capture(tok_dev, warmup=1)
    eng.replay()
    torch.cuda.synchronize()
    with ClockSampler(dev.index) as clk:
        ms = time_graph(eng, args.steps, dist)
    sparsity = achieved_sparsity(eng, model)
    # e2e through the public API: host (pinned) batch -> device, step, loss -> host, every step
    pinned = [b.pin_memory() for b in batches]
    loss_host = torch.empty((), dtype=torch.float32).pin_memory()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st.record()
    for k in range(args.steps):
        loss = eng.replay(pinned[k % len(pinned)])
        loss_host.copy_(loss, non_blocking=True)
    en.record()
    torch.cuda.synchronize()
    e2e_ms = st.elapsed_time(en) / args.steps
    if dist is not None:
        t = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    final_loss = float(loss_host)
    roof = fc1_roofline(model, eng, tok_dev, peaks, args.config) if rank == 0 else None
    frozen_gb = sum(t.numel() * t.element_size() for lw in model.weights.layers
                    for t in (lw.wqkv, lw.wo, lw.mlp.w1_t, lw.mlp.w2)) / 1e9
    extra = {}
    if not args.skip_dense and rank == 0:
        # dense reference points on the same box: (a) same engine, every head/block dense; (b) torch cuBLAS/SDPA
        dprov = HN.DenseProvider(model)
        deng = FinetuneEngine(model, state, dprov, lr=1e-4)
        deng.step(tok_dev)
        deng.capture(tok_dev, warmup=1)
        extra["dense_same_kernels_ms"] = round(time_graph(deng, max(3, args.steps // 2), None), 3)
        del deng
        torch.cuda.empty_cache()
        try:
            tstep = DenseLoraStep(model)
            for _ in range(2):
                tstep.step(tok_dev)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            n = max(3, args.steps // 2)
            for _ in range(n):
                tstep.step(tok_dev)
            b.record()
            torch.cuda.synchronize()
            extra["dense_torch_ms"] = round(a.elapsed_time(b) / n, 3)
            extra["speedup_vs_dense_torch"] = round(extra["dense_torch_ms"] / ms, 3)
            del tstep
        except Exception as e:  # pragma: no cover
            extra["dense_torch_error"] = repr(e)[:200]
    cpu = None
    if rank == 0 and world == 1 and not args.skip_cpu:
        cpu = cpu_baseline(cfg, args)
    tokens_per_step = B * s * world
    line = {
        "metric": f"{cfg['desc']} LoRA fwd+bwd ms/batch", "value": round(ms, 3), "unit": "ms/batch", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": False,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic (uniform tokens, random-init weights)",
        "config": {"workload": f"{args.config}: {cfg['desc']} LoRA r={cfg['r']} (wq,wv,w1,w2) fine-tune step (predict+fwd+bwd+Adam), predicted mode",
                   "model": cfg["desc"], "global_batch": B * world, "seq_len": s, "parallelism": f"dp{world}",
                   "d_model": cfg["d"], "n_layers": cfg["L"], "d_ff": cfg["d_ff"], "vocab": V, "blk_size": cfg["blk"],
                   "attn_blk": cfg["attn_blk"], "mask_scope": "per sequence", **sparsity,
                   "injected": {"mlp_zeroed_predictor_blocks": args.mlp_sparsity, "local_attention_heads": args.local_frac},
                   "l2": f"inputs larger than L2: {frozen_gb:.1f} GB of frozen weights stream from HBM every step (no flush needed)",
                   "timing": "CUDA events around K CUDA-graph replays; Adam (fp64 moments) outside the graph, inside the timed region"},
        "tokens_per_s": round(tokens_per_step / (ms * 1e-3), 1),
        "e2e": {"value": round(e2e_ms, 3), "unit": "ms/batch", "h2d_bytes_per_step": int(B * (s + 1) * 8),
                "d2h_bytes_per_step": 4, "api": "FinetuneEngine.replay(host pinned batch) + loss.copy_ to host"},
        "gpu_launches": int(per_step * args.steps), "gpu_launches_per_step": int(per_step),
        "final_loss": round(final_loss, 5),
        "clocks": clk.summary(),
        "roofline": roof,
        "cpu_baseline": cpu,
        **extra,
    }
    return line


# ---------------------------------------------------------------------------- CPU reference (oracle port)


def cpu_baseline(cfg: dict, args, n_layers_sample: int = 2) -> dict:
    """Time the reference algorithm (oracle/ NumPy restatement of sf/harness.py:401-417) on the host
    cores on a bounded sample — one sequence through `n_layers_sample` layers + LM head + Adam — and
    extrapolate to the full batch (B sequences, L layers)."""
    from oracle import sf_oracle as O

    try:
        from threadpoolctl import threadpool_info

        blas_threads = max((i.get("num_threads", 1) for i in threadpool_info()), default=1)
    except Exception:  # pragma: no cover
        blas_threads = os.cpu_count()
    d, H, f, s, V = cfg["d"], cfg["H"], cfg["d_ff"], cfg["s"], cfg["V"]
    dims = O.Dims(d, H, f, s, n_layers_sample, V, cfg["blk"], cfg["attn_blk"])
    om = O.build_model(dims, seed=args.seed, peft="lora", lora_rank=cfg["r"])
    rng = O.make_rng(args.seed + 1)
    n_blk = dims.n_blk
    r_pred = max(4, d // 16)
    attn, mlp = [], []
    n_local = int(round(H * args.local_frac))
    for layer in range(n_layers_sample):
        wq = [O.randn(rng, (d, r_pred), 0.1) for _ in range(H)]
        wk = [wq[h] if h < n_local else O.randn(rng, (d, r_pred), 0.1) for h in range(H)]
        attn.append(O.AttnPredictorParams(wq, wk))
        wa = O.randn(rng, (d, n_blk), 0.1)
        wa[:, rng.permutation(n_blk)[: int(round(args.mlp_sparsity * n_blk))]] = 0.0
        mlp.append(O.MlpPredictorParams(wa))
    prov = O.PredictedProvider(om, attn, mlp, O.PredictorConfig())
    seq = rng.integers(0, V, size=s + 1)
    tok, tgt = seq[:-1], seq[1:]
    params = O.trainable_params(om)

    def one():
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
        return t

    one()  # warm-up
    runs = [one() for _ in range(2)]
    med = {k: statistics.median(r[k] for r in runs) for k in runs[0]}
    per_layer = (med["layers_fwd"] + med["layers_bwd"]) / n_layers_sample
    per_item = per_layer * cfg["L"] + med["head"]
    adam_full = med["adam"] * cfg["L"] / n_layers_sample
    batch_s = cfg["B"] * per_item + adam_full
    return {"value": round(batch_s * 1e3, 1), "unit": "ms/batch", "cores": int(blas_threads), "kind": "port",
            "sample": (f"1 sequence x {n_layers_sample} of {cfg['L']} layers + LM head + Adam on the oracle "
                       f"(NumPy restatement of sf/harness.py:401-417, predicted mode, same injected sparsity), "
                       f"extrapolated x{cfg['B']} sequences x{cfg['L']}/{n_layers_sample} layers; "
                       f"measured per-layer {per_layer * 1e3:.0f} ms, head {med['head'] * 1e3:.0f} ms"),
            "host_cpu_count": os.cpu_count()}


def run_reference(args, cfg, rank) -> dict | None:
    if rank != 0:
        return None
    cpu = cpu_baseline(cfg, args)
    return {"impl": "reference", "metric": f"{cfg['desc']} LoRA fwd+bwd ms/batch", "value": cpu["value"], "unit": "ms/batch",
            "n_gpus": int(os.environ.get("WORLD_SIZE", 1)), "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": cpu["value"], "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "config": {"workload": "cfg3 (as ours), reference algorithm on host cores", "model": cfg["desc"],
                                            "global_batch": cfg["B"], "seq_len": cfg["s"], "parallelism": "host"},
            "cpu_baseline": cpu, "e2e": {"value": cpu["value"], "unit": "ms/batch", "h2d_bytes_per_step": 0,
                                         "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg3", choices=sorted(CONFIGS))
    ap.add_argument("--mlp-sparsity", type=float, default=0.85)
    ap.add_argument("--local-frac", type=float, default=0.5)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--batch", type=int, default=0, help="sequences per rank (default: the config's B)")
    ap.add_argument("--skip-dense", action="store_true")
    ap.add_argument("--skip-cpu", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    cfg = dict(CONFIGS[args.config])
    if args.batch:
        cfg["B"] = args.batch
    world = int(os.environ.get("WORLD_SIZE", 1))
    rank = int(os.environ.get("RANK", 0))
    if args.impl == "reference":
        line = run_reference(args, cfg, rank)
        if line is not None:
            print(json.dumps(line), flush=True)
        return
    dist = None
    if world > 1:
        import torch
        import torch.distributed as tdist

        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)) % max(torch.cuda.device_count(), 1))
        # NCCL over NVLink in production; LX_DIST_BACKEND=gloo lets several ranks share one GPU (plumbing checks)
        tdist.init_process_group(os.environ.get("LX_DIST_BACKEND", "nccl"))
        dist = tdist
    line = run_ours(args, cfg, rank, world, dist)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
