#!/usr/bin/env python
"""Offline pipeline and oracle-mode timings at cfg3 (OPT-1.3B shapes, s = 512) on one B200.

* collect-traces (compact form) for --traces sequences, batch 8: wall time incl. the host copies
  and the .tnsc write (it is an offline job);
* train-predictors for --layers layers with the reference defaults (200 epochs, noise 0.05,
  rank d/16 = 128, recall weight 4): wall time per layer;
* fine-tune step (B = 8) under the exposer-oracle and shadowy providers (dense ground-truth masks)
  next to the predicted provider, device time per step (CUDA events, eager engine, 3 warm-up).

    python tools/offline_bench.py [--traces 10] [--layers 2] [--steps 3]
"""

from __future__ import annotations

import argparse
import json
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--traces", type=int, default=10)
    ap.add_argument("--layers", type=int, default=2)
    ap.add_argument("--steps", type=int, default=3)
    args = ap.parse_args()
    import torch

    from bench import CONFIGS, build_workload
    from paper_2510_15964_b200 import engine as EN, harness as HN, offline as OF, predictor as P

    cfg = dict(CONFIGS["cfg3"])
    dev = torch.device("cuda")
    model, state, pred_provider = build_workload(cfg, dev, seed=0, mlp_sparsity=0.5, local_frac=0.5)
    dims = model.dims
    corpus = np.random.default_rng(1).integers(0, dims.vocab, size=(args.traces, dims.seq_len))
    with tempfile.TemporaryDirectory() as td:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        tens = OF.collect_traces(model, corpus, Path(td) / "traces.tnsc", batch=8)
        t_collect = time.perf_counter() - t0
        size = (Path(td) / "traces.tnsc").stat().st_size
        traces = OF.load_traces(tens, dims.n_layers, dims.n_heads, dims.blk_size)
    print(json.dumps({"phase": "collect_traces", "traces": args.traces, "s": dims.seq_len, "layers": dims.n_layers,
                      "seconds": round(t_collect, 3), "file_mb": round(size / 2**20, 1),
                      "full_form_mb_estimate": round(args.traces * dims.n_layers * (2 * dims.n_heads * dims.seq_len**2 * 8
                                                     + dims.seq_len * (2 * dims.d_model + dims.d_ff) * 4) / 2**20, 1)}),
          flush=True)
    pcfg = P.PredictorTrainConfig()
    n_train = max(1, int(0.8 * len(traces)))
    train = traces[:n_train]
    for layer in range(args.layers):
        ap_ = OF.init_attn_predictor(dims.d_model, dims.n_heads, seed=100 + layer)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        la = OF.train_attn_predictor([t[layer]["x_attn_ds"] for t in train], [t[layer]["raw_ds"] for t in train], ap_, pcfg,
                                     seed=200 + layer)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        mp = OF.init_mlp_predictor(dims.d_model, dims.n_blk, seed=300 + layer)
        lm = OF.train_mlp_predictor([t[layer]["x_mlp"] for t in train], [t[layer]["active_bits"] for t in train],
                                    dims.n_blk, mp, pcfg, seed=400 + layer)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        print(json.dumps({"phase": "train_predictors", "layer": layer, "epochs": pcfg.epochs, "train_traces": n_train,
                          "attn_seconds": round(t1 - t0, 3), "mlp_seconds": round(t2 - t1, 3), "attn_loss": la,
                          "mlp_loss": lm}), flush=True)
    B = cfg["B"]
    tok = torch.as_tensor(np.random.default_rng(2).integers(0, dims.vocab, size=(B, dims.seq_len + 1)), device=dev)
    for name, prov in (("predicted", pred_provider), ("exposer-oracle", HN.OracleProvider(model, theta=0.1, tau=0.95)),
                       ("shadowy", HN.ShadowyProvider(model, tau=0.95))):
        prov.timing = False
        eng = EN.FinetuneEngine(model, state, prov, lr=1e-4)
        for _ in range(3):
            eng.step(tok)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(args.steps):
            eng.step(tok)
        b.record()
        b.synchronize()
        ms = a.elapsed_time(b) / args.steps
        masks = eng.last_masks
        act = float(np.mean([lm.neuron_mask.counts.float().mean().item() / dims.n_blk for lm in masks]))
        print(json.dumps({"phase": "finetune_step", "provider": name, "B": B, "ms_per_step_eager": round(ms, 2),
                          "mlp_active_frac": round(act, 3)}), flush=True)


if __name__ == "__main__":
    main()
