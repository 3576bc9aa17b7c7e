"""GPU parity of the offline predictor pipeline (offline.py, csrc/offline.cu) against the
reference's own training runs (tests/golden/offline.npz, oracle/make_golden_offline.py).

Bars: truth labels are bit work — bit-exact. Training without input noise is
deterministic on both sides: the loss within 1e-4 relative and 99% of the trained
weights within 1e-4 absolute (fp32 GEMM rounding only; an entry whose gradient is
~0 may take a different Adam sign, hence the quantile). With noise the draws differ
(torch vs NumPy generators): final loss within 25% of the reference's."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    return torch.device("cuda")


def test_truth_labels_bit_exact(dev, golden):
    from paper_2510_15964_b200 import offline as OF

    g = golden("offline")
    d, s, d_ff, blk, n = (int(v) for v in g["m/meta"])
    for i in range(n):
        bits = OF.mlp_truth_labels(torch.from_numpy(g[f"m/z{i}"]).to(dev), blk)
        np.testing.assert_array_equal(OF.bits_to_bool(bits, -(-d_ff // blk)).cpu().numpy(), g[f"m/labels{i}"])
    z, blk = g["lab/z"], int(g["lab/blk"])
    bits = OF.mlp_truth_labels(torch.from_numpy(z).to(dev), blk)
    np.testing.assert_array_equal(OF.bits_to_bool(bits, -(-z.shape[1] // blk)).cpu().numpy(), g["lab/labels"])


@pytest.mark.parametrize("blk,n_cols", [(1, 70), (16, 8192), (7, 100), (64, 1000)])
def test_truth_labels_shapes(dev, blk, n_cols):
    from paper_2510_15964_b200 import offline as OF

    rng = np.random.default_rng(blk + n_cols)
    z = (rng.standard_normal((33, n_cols)) - 2.0).astype(np.float32)
    n_blk = -(-n_cols // blk)
    want = np.stack([np.array([(z[t, b * blk : (b + 1) * blk] > 0).any() for b in range(n_blk)]) for t in range(33)])
    got = OF.bits_to_bool(OF.mlp_truth_labels(torch.from_numpy(z).to(dev), blk), n_blk).cpu().numpy()
    np.testing.assert_array_equal(got, want)


def _close(got, ref, noise):
    if noise:
        return
    dlt = np.abs(np.asarray(got, np.float64) - ref)
    assert np.quantile(dlt, 0.99) < 1e-4, dlt.max()


@pytest.mark.parametrize("tag", ["a0", "a1"])
def test_train_attn_predictor_matches_reference(dev, golden, tag):
    from paper_2510_15964_b200 import offline as OF, predictor as P

    g = golden("offline")
    d, H, r, s, n, noise, epochs, lr = g[f"{tag}/meta"]
    H, n = int(H), int(n)
    params = P.AttnPredictorParams(list(g[f"{tag}/wq0"]), list(g[f"{tag}/wk0"]))
    cfg = P.PredictorTrainConfig(noise_std=float(noise), epochs=int(epochs), lr=float(lr))
    xs = [g[f"a/x{i}"] for i in range(n)]
    raws = [[g[f"a/raw{i}.{h}"] for h in range(H)] for i in range(n)]
    loss = OF.train_attn_predictor(xs, raws, params, cfg, seed=9, device=dev)
    ref = float(g[f"{tag}/loss"])
    assert abs(loss - ref) <= (0.25 if noise else 1e-4) * ref, (loss, ref)
    _close(np.stack(params.wq_hat), g[f"{tag}/wq"], noise)
    _close(np.stack(params.wk_hat), g[f"{tag}/wk"], noise)


@pytest.mark.parametrize("tag", ["m0", "m1"])
def test_train_mlp_predictor_matches_reference(dev, golden, tag):
    from paper_2510_15964_b200 import offline as OF, predictor as P

    g = golden("offline")
    d, s, d_ff, blk, n = (int(v) for v in g["m/meta"])
    noise = 0.0 if tag == "m0" else 0.05
    params = P.MlpPredictorParams(g[f"{tag}/wa0"].copy())
    cfg = P.PredictorTrainConfig(noise_std=noise, epochs=25, lr=1e-2, recall_weight=4.0)
    bits = [OF.mlp_truth_labels(torch.from_numpy(g[f"m/z{i}"]).to(dev), blk) for i in range(n)]
    loss = OF.train_mlp_predictor([g[f"m/x{i}"] for i in range(n)], bits, -(-d_ff // blk), params, cfg, seed=11, device=dev)
    ref = float(g[f"{tag}/loss"])
    assert abs(loss - ref) <= (0.25 if noise else 1e-4) * ref, (loss, ref)
    _close(params.wa_hat, g[f"{tag}/wa"], noise)


def test_collect_train_roundtrip(dev, tmp_path):
    """collect-traces -> train-predictors -> predicted-mode step, through .tnsc files; the compact
    trace form carries the same training inputs as the reference-compatible full form."""
    from oracle import sf_oracle as O
    from paper_2510_15964_b200 import harness as HN, model as M, offline as OF, predictor as P, tnsc

    om = O.build_model(O.Dims(64, 2, 128, 64, 2, 80, 16, 16), seed=3, peft="lora")
    d = om.dims
    dims = M.ModelDims(d.d_model, d.n_heads, d.d_ff, d.seq_len, d.n_layers, d.vocab, d.blk_size, d.attn_blk)
    m = M.from_arrays(dims, om.peft, om.emb, om.layers, om.lnf_g, om.lnf_b, lora=om.lora, lora_targets=om.lora_targets,
                      device=dev)
    corpus = np.random.default_rng(4).integers(0, dims.vocab, size=(5, dims.seq_len))
    OF.collect_traces(m, corpus, tmp_path / "traces.tnsc", batch=3)
    full = OF.collect_traces(m, corpus[:2], tmp_path / "full.tnsc", batch=2, full=True)
    assert f"trace1.layer1.probs.h{dims.n_heads - 1}" in full and "trace0.layer0.z" in full
    tc = OF.load_traces(tmp_path / "traces.tnsc", dims.n_layers, dims.n_heads, dims.blk_size, device=dev)
    tf = OF.load_traces(tmp_path / "full.tnsc", dims.n_layers, dims.n_heads, dims.blk_size, device=dev)
    assert len(tc) == 5 and len(tf) == 2
    for i in range(2):
        for layer in range(dims.n_layers):
            a, b = tc[i][layer], tf[i][layer]
            np.testing.assert_array_equal(a["x_attn_ds"], b["x_attn_ds"])
            np.testing.assert_array_equal(a["x_mlp"], b["x_mlp"])
            for h in range(dims.n_heads):
                np.testing.assert_allclose(a["raw_ds"][h], b["raw_ds"][h], rtol=1e-5, atol=1e-6)
            np.testing.assert_array_equal(np.asarray(a["active_bits"]), np.asarray(b["active_bits"]))
    cfg = P.PredictorTrainConfig(epochs=30, lr=1e-2)
    preds, metrics = OF.train_predictors(m, tc, cfg, rank=8, seed=0, out_path=tmp_path / "pred.tnsc")
    assert all(np.isfinite(metrics["attn_final_loss"])) and all(np.isfinite(metrics["mlp_final_loss"]))
    assert 0.0 <= metrics["attn_pattern_agreement"] <= 1.0 and 0.0 <= metrics["mlp_recall"] <= 1.0
    back = OF.load_predictors(tmp_path / "pred.tnsc", dims.n_layers, dims.n_heads)
    np.testing.assert_array_equal(back["mlp"][1].wa_hat, preds["mlp"][1].wa_hat)
    t, _ = tnsc.load_tensors(tmp_path / "pred.tnsc")
    assert f"layers.1.attn.h{dims.n_heads - 1}.wk_hat" in t
    prov = HN.PredictedProvider(m, back, cfg)
    out = HN.finetune_step(m, M.make_peft_state(m), np.random.default_rng(5).integers(0, dims.vocab, (2, dims.seq_len + 1)),
                           prov, lr=1e-3)
    assert np.isfinite(out["loss"])
