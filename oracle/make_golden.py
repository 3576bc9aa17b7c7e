"""TEST INFRASTRUCTURE ONLY — generate tests/golden/*.npz from the UNMODIFIED
reference (`sparseft`, imported from /root/reference/pkg/src).

Run in the build container (the reference does not exist on the GPU box):

    python oracle/make_golden.py

Every fixture stores the reference's own inputs and outputs; the oracle
(`oracle/sf_oracle.py`) is pinned against them by tests/test_oracle_golden.py
and the GPU path by tests/test_gpu_*.py.
"""

from __future__ import annotations

import hashlib
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"


def _h(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main() -> None:
    sys.path.insert(0, str(REF))
    from sparseft import autograd, bench, block_sparse as BS, exposer as E, model as M, neuron_ops as N  # noqa: E402
    from sparseft import patterns as PT, predictor as P  # noqa: E402
    from sparseft.tensor_core import make_rng  # noqa: E402

    OUT.mkdir(parents=True, exist_ok=True)
    rng = make_rng(1234)

    # ---- pattern pools ---------------------------------------------------
    pools = {}
    for n_b in (2, 3, 4, 5, 8, 16, 32):
        for pid, t in PT.build_pool(n_b).items():
            pools[f"n{n_b}/{pid}"] = np.asarray(t.coords, dtype=np.int32).reshape(-1, 2)
        pools[f"n{n_b}/__order__"] = np.array(list(PT.build_pool(n_b)), dtype="U16")
    np.savez_compressed(OUT / "pools.npz", **pools)

    # ---- predictor / exposer mask logic on given scores ------------------
    pred = {}
    pred["ds_s"] = np.array([1, 2, 7, 10, 16, 64, 100, 256, 512, 1000, 1024, 2048])
    for s in pred["ds_s"]:
        pred[f"ds/{s}"] = P.downsample_indices(int(s))
    cases = []
    for c in range(60):
        m = int(rng.integers(2, 34))
        n_b = int(rng.choice([2, 3, 4, 8, 16, 32]))
        frac = float(rng.choice([0.5, 0.3, 0.75, 0.9]))
        tau = float(rng.choice([0.9, 0.95, 0.5, 1.0]))
        kind = c % 4
        if kind == 0:
            s_hat = rng.standard_normal((m, m)).astype(np.float32)
        elif kind == 1:  # gram-like, diagonal dominant
            x = rng.standard_normal((m, 16)).astype(np.float32)
            s_hat = (x @ x.T).astype(np.float32)
        elif kind == 2:  # all negative -> all-false grid -> dense
            s_hat = -np.abs(rng.standard_normal((m, m))).astype(np.float32) - 0.1
        else:  # banded
            i = np.arange(m)
            s_hat = (np.exp(-np.abs(i[:, None] - i[None, :]).astype(np.float32)) + 0.01 * rng.standard_normal((m, m))).astype(np.float32)
        pool = PT.build_pool(n_b)
        cell = P.binarize_scores(s_hat, frac)
        grid = P.upsample_mask(cell, n_b).astype(np.float64)
        pid = E.select_pattern_by_coverage(grid, pool, tau)
        pred[f"case{c}/s_hat"] = s_hat
        pred[f"case{c}/meta"] = np.array([m, n_b, frac, tau])
        pred[f"case{c}/cell"] = cell
        pred[f"case{c}/grid"] = grid
        pred[f"case{c}/pid"] = np.array(pid)
        cases.append(c)
    pred["n_cases"] = np.array(len(cases))
    # float grids (oracle-mode coverage)
    for c in range(30):
        n_b = int(rng.choice([2, 4, 8]))
        g = np.abs(rng.standard_normal((n_b, n_b))) + (np.eye(n_b) * rng.uniform(0, 20))
        tau = float(rng.choice([0.5, 0.8, 0.95, 0.99]))
        pred[f"fgrid{c}/g"] = g
        pred[f"fgrid{c}/tau"] = np.array(tau)
        pred[f"fgrid{c}/pid"] = np.array(E.select_pattern_by_coverage(g, PT.build_pool(n_b), tau))
    # MLP mask prediction
    for c in range(12):
        s, n_blk, nb = int(rng.integers(1, 40)), int(rng.integers(1, 70)), int(rng.integers(1, 4))
        thr = float(rng.choice([0.0, 0.5, -0.2]))
        shat = [(rng.standard_normal((s, n_blk)) - 1.5).astype(np.float32) for _ in range(nb)]
        for j, a in enumerate(shat):
            pred[f"mlp{c}/s{j}"] = a
        pred[f"mlp{c}/meta"] = np.array([nb, thr])
        pred[f"mlp{c}/mask"] = P.predict_mlp_mask(shat, thr)
    # importance + theta filter
    for c in range(8):
        z = rng.standard_normal((int(rng.integers(1, 20)), int(rng.integers(1, 80)))).astype(np.float32)
        blk = int(rng.choice([1, 4, 16]))
        th = float(rng.choice([0.0, 0.1, 0.5, 1.0]))
        imp = E.block_importance(z, blk)
        pred[f"imp{c}/z"] = z
        pred[f"imp{c}/meta"] = np.array([blk, th])
        pred[f"imp{c}/imp"] = imp
        pred[f"imp{c}/mask"] = E.filter_neuron_blocks(imp, th)
    # end-to-end predict_attention_patterns with real low-rank factors
    for c in range(6):
        d, H, r, s, n_b = 64, 3, 8, int(rng.choice([64, 100, 128])), int(rng.choice([4, 8]))
        if s % n_b:
            s = n_b * (s // n_b)
        params = P.init_attn_predictor(d, H, rank=r, seed=c)
        if c % 2:
            params.wk_hat = [w.copy() for w in params.wq_hat]  # gram -> diagonal heads
        xb = [rng.standard_normal((s, d)).astype(np.float32) for _ in range(1 + c % 2)]
        out = P.predict_attention_patterns(xb, params, PT.build_pool(n_b), P.PredictorTrainConfig())
        pred[f"pap{c}/wq"] = np.stack(params.wq_hat)
        pred[f"pap{c}/wk"] = np.stack(params.wk_hat)
        for j, x in enumerate(xb):
            pred[f"pap{c}/x{j}"] = x
        pred[f"pap{c}/meta"] = np.array([len(xb), n_b])
        pred[f"pap{c}/out"] = np.array(out)
    np.savez_compressed(OUT / "predictor.npz", **pred)

    # ---- block-sparse operators -----------------------------------------
    bs = {}
    for c, (s, hd, blk, sp) in enumerate([(64, 32, 16, 0.5), (128, 64, 16, 0.75), (128, 64, 32, 0.0), (256, 64, 64, 0.5), (128, 128, 16, 0.9)]):
        n_b = s // blk
        q, k, v, do = (rng.standard_normal((s, hd)).astype(np.float32) for _ in range(4))
        coords = bench._attn_layout(n_b, sp, rng)
        scale = 1.0 / np.sqrt(hd)
        sc = BS.sdd(q, k, coords, blk, scale)
        p = BS.sparse_softmax(sc)
        o = BS.dsd(p, v)
        db, dv = BS.dsd_backward(p, v, do)
        ds = BS.sparse_softmax_backward(p, db)
        dq, dk = BS.sdd_backward(ds, q, k, p.coords, blk, scale)
        for n, a in dict(q=q, k=k, v=v, do=do, coords=np.array(coords, np.int32), scores=sc.blocks, probs=p.blocks, out=o,
                         d_blocks=db, dv=dv, ds=ds, dq=dq, dk=dk, meta=np.array([s, hd, blk]),
                         dense=BS.dense_masked_attention(q, k, v, coords, blk, scale)).items():
            bs[f"c{c}/{n}"] = a
    bs["n_cases"] = np.array(5)
    np.savez_compressed(OUT / "block_sparse.npz", **bs)

    # ---- neuron ops --------------------------------------------------------
    no = {}
    for c, (s, d, d_ff, blk, sp) in enumerate([(32, 64, 256, 16, 0.5), (64, 128, 512, 16, 0.9), (16, 64, 200, 16, 0.3), (16, 32, 64, 16, 1.0)]):
        x = rng.standard_normal((s, d)).astype(np.float32)
        w1 = rng.standard_normal((d, d_ff)).astype(np.float32)
        w2 = rng.standard_normal((d_ff, d)).astype(np.float32)
        nb = N.n_blocks(d_ff, blk)
        mask = bench._spread_mask(nb, sp) if sp < 1.0 else np.zeros(nb, bool)
        lw = N.LayeredWeights.from_row_major(w1, w2)
        hid = N.neuron_matmul_fwd1(x, lw, mask, blk)
        hid2 = N.ActiveHidden(np.maximum(hid.values, 0), hid.active_blocks, hid.col_index, blk, d_ff)
        out = N.neuron_matmul_fwd2(hid2, lw, mask)
        for n, a in dict(x=x, w1=w1, w2=w2, mask=mask, cols=hid.col_index, h=hid.values, out=out, meta=np.array([blk])).items():
            no[f"c{c}/{n}"] = a
    no["n_cases"] = np.array(4)
    np.savez_compressed(OUT / "neuron_ops.npz", **no)

    # ---- model forward / backward / Adam (float32, tiny dims) ------------
    md = {}
    dims = M.ModelDims(d_model=128, n_heads=2, d_ff=256, seq_len=64, n_layers=2, vocab=96, blk_size=16, attn_blk=16)
    md["dims"] = np.array([128, 2, 256, 64, 2, 96, 16, 16])
    for peft in ("lora", "adapter", "bitfit"):
        model = M.build_model(dims, seed=7, peft=peft)
        r2 = make_rng(99)
        for ad in model.lora.values():
            ad.b += (r2.standard_normal(ad.b.shape) * 0.02).astype(np.float32)
        for ad in model.adapters.values():
            ad.w_up += (r2.standard_normal(ad.w_up.shape) * 0.02).astype(np.float32)
        if peft == "bitfit":
            for lw in model.weights.layers:
                for b in M.BIAS_NAMES:
                    getattr(lw, b)[...] += (r2.standard_normal(getattr(lw, b).shape) * 0.02).astype(np.float32)
        # weight fingerprints (pin the oracle's build_model draw order)
        md[f"{peft}/hash_w1_l1"] = np.array(_h(model.weights.layers[1].mlp.w1.T))  # [d_ff, d] row-major bytes
        md[f"{peft}/hash_emb"] = np.array(_h(model.weights.emb))
        for name, p in M.trainable_params(model).items():
            md[f"{peft}/param/{name}"] = p.copy()
        toks = r2.integers(0, dims.vocab, size=dims.seq_len + 1)
        masks = []
        pids = list(model.pool)
        for i in range(dims.n_layers):
            hp = [pids[int(r2.integers(len(pids)))] for _ in range(dims.n_heads)]
            nm = r2.random(dims.n_blk) < 0.6
            nm[0] = True
            masks.append(M.LayerMasks(hp, nm))
            md[f"{peft}/masks/{i}/heads"] = np.array(hp)
            md[f"{peft}/masks/{i}/neuron"] = nm
        logits, cache = M.model_forward(model, toks[:-1], masks)
        loss = M.loss_forward(logits, toks[1:])
        grads = autograd.model_backward(model, cache, M.loss_backward(logits, toks[1:]), masks)
        md[f"{peft}/tokens"] = toks
        md[f"{peft}/logits"] = logits
        md[f"{peft}/loss"] = np.array(loss)
        for i in range(dims.n_layers):
            md[f"{peft}/h_out/{i}"] = cache["blocks"][i]["mlp"]["x"]  # post-LN2 MLP input
        for n, g in grads.items():
            md[f"{peft}/grad/{n}"] = g
        state = M.make_peft_state(model)
        autograd.optimizer_step(state, grads, lr=1e-3)
        for n, p in state.params.items():
            md[f"{peft}/after_adam/{n}"] = p.copy()
    np.savez_compressed(OUT / "model.npz", **md)

    # ---- one predicted-mode fine-tune step (harness semantics) ------------
    from sparseft import harness as HN

    ft = {}
    dims = M.ModelDims(d_model=128, n_heads=2, d_ff=256, seq_len=64, n_layers=2, vocab=96, blk_size=16, attn_blk=16)
    model = M.build_model(dims, seed=3, peft="lora")
    cfg = HN.RunConfig(d_model=128, n_heads=2, d_ff=256, seq_len=64, n_layers=2, vocab=96, mode="predicted", batch_size=2)
    attn = [P.init_attn_predictor(128, 2, rank=8, seed=10 + i) for i in range(2)]
    attn[1].wk_hat = [w.copy() for w in attn[1].wq_hat]
    mlp = [P.init_mlp_predictor(128, dims.n_blk, seed=20 + i) for i in range(2)]
    for i in range(2):
        mlp[i].wa_hat[:, ::3] = 0.0  # zero columns -> never active (sparsity injection)
    prov = HN.PredictedProvider(model, {"attn": attn, "mlp": mlp}, cfg)
    r3 = make_rng(5)
    batch = r3.integers(0, 96, size=(2, 65))
    state = M.make_peft_state(model)
    gsum, losses, pats, nmasks = {}, [], [], []
    for seq in batch:
        logits, cache = M.model_forward(model, seq[:-1], prov)
        losses.append(M.loss_forward(logits, seq[1:]))
        ms = [c["masks"] for c in cache["blocks"]]
        pats.append([m.head_patterns for m in ms])
        nmasks.append([m.neuron_mask for m in ms])
        g = autograd.model_backward(model, cache, M.loss_backward(logits, seq[1:]), ms)
        for n, v in g.items():
            gsum[n] = gsum.get(n, 0) + v
    gmean = {n: v / 2 for n, v in gsum.items()}
    autograd.optimizer_step(state, gmean, lr=1e-3)
    ft["batch"] = batch
    ft["loss"] = np.array(np.mean(losses))
    ft["patterns"] = np.array(pats)
    ft["neuron_masks"] = np.array(nmasks)
    for i in range(2):
        ft[f"attn{i}/wq"] = np.stack(attn[i].wq_hat)
        ft[f"attn{i}/wk"] = np.stack(attn[i].wk_hat)
        ft[f"mlp{i}/wa"] = mlp[i].wa_hat
    for n, v in gmean.items():
        ft[f"grad/{n}"] = v
    for n, p in state.params.items():
        ft[f"after/{n}"] = p.copy()
    np.savez_compressed(OUT / "finetune_step.npz", **ft)
    for f in sorted(OUT.glob("*.npz")):
        print(f.name, f.stat().st_size)


if __name__ == "__main__":
    main()
