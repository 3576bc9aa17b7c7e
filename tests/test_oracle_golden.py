"""Pin the CPU oracle (oracle/sf_oracle.py) against the reference's golden
vectors (tests/golden, produced by oracle/make_golden.py from the unmodified
reference) and against the reference's own known-answer tests
(pkg/tests/test_patterns.py, test_predictor.py, test_exposer.py,
test_block_sparse.py, test_neuron_ops.py, test_autograd.py)."""

import hashlib

import numpy as np
import pytest

from oracle import sf_oracle as O


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-30)


# ---------------------------------------------------------------- patterns
def test_pools_match_reference(golden):
    g = golden("pools")
    for n_b in (2, 3, 4, 5, 8, 16, 32):
        pool = O.build_pool(n_b)
        assert list(pool) == list(g[f"n{n_b}/__order__"])
        for pid, c in pool.items():
            np.testing.assert_array_equal(c, g[f"n{n_b}/{pid}"])


def test_pool_kats():
    # pkg/tests/test_patterns.py:10-60
    p = O.build_pool(4)
    assert list(p) == ["blockdiag", "band1", "band2", "causal1", "global1", "strided2", "dense"]
    assert len(p["band1"]) == 10 and len(p["causal1"]) == 7
    with pytest.raises(O.PatternError):
        O.build_pool(2, band_widths=(3,))
    with pytest.raises(O.PatternError):
        O.build_pool(0)
    ent, off = O.combine_layouts(["blockdiag", "blockdiag"], O.build_pool(4))
    assert tuple(off) == (0, 4) and ent.shape == (8, 3)
    with pytest.raises(O.PatternError):
        O.combine_layouts(["nope"], O.build_pool(4))


# ---------------------------------------------------------------- predictor
def test_downsample_indices(golden):
    g = golden("predictor")
    for s in g["ds_s"]:
        np.testing.assert_array_equal(O.downsample_indices(int(s)), g[f"ds/{s}"])
    np.testing.assert_array_equal(O.downsample_indices(16), [0, 4, 8, 12])


def test_binarize_upsample_select_bit_exact(golden):
    g = golden("predictor")
    for c in range(int(g["n_cases"])):
        s_hat = g[f"case{c}/s_hat"]
        m, n_b, frac, tau = g[f"case{c}/meta"]
        cell = O.binarize_scores(s_hat, float(frac))
        np.testing.assert_array_equal(cell, g[f"case{c}/cell"])
        grid = O.upsample_mask(cell, int(n_b)).astype(np.float64)
        np.testing.assert_array_equal(grid, g[f"case{c}/grid"])
        assert O.select_pattern_by_coverage(grid, O.build_pool(int(n_b)), float(tau)) == str(g[f"case{c}/pid"])


def test_select_float_grids(golden):
    g = golden("predictor")
    for c in range(30):
        grid = g[f"fgrid{c}/g"]
        pid = O.select_pattern_by_coverage(grid, O.build_pool(grid.shape[0]), float(g[f"fgrid{c}/tau"]))
        assert pid == str(g[f"fgrid{c}/pid"])


def test_select_kats():
    # pkg/tests/test_exposer.py:99-133
    pool = O.build_pool(4)
    assert O.select_pattern_by_coverage(np.eye(4) * 10.0 + 0.01, pool, 0.95) == "blockdiag"
    assert O.select_pattern_by_coverage(np.ones((4, 4)), pool, 0.99) == "dense"
    band = np.array([[abs(i - j) <= 1 for j in range(4)] for i in range(4)], float)
    assert O.select_pattern_by_coverage(band, pool, 0.99) == "band1"
    assert O.select_pattern_by_coverage(np.zeros((4, 4)), pool, 0.95) == "dense"
    with pytest.raises(ValueError):
        O.select_pattern_by_coverage(np.ones((4, 4)), pool, 0.0)


def test_binarize_kats():
    np.testing.assert_array_equal(O.binarize_scores(np.array([[10.0, 6.0], [4.0, 1.0]]), 0.5), [[True, True], [False, False]])
    np.testing.assert_array_equal(O.binarize_scores(np.array([[10.0, 5.0]]), 0.5), [[True, False]])


def test_mlp_mask(golden):
    g = golden("predictor")
    for c in range(12):
        nb, thr = g[f"mlp{c}/meta"]
        shat = [g[f"mlp{c}/s{j}"] for j in range(int(nb))]
        np.testing.assert_array_equal(O.predict_mlp_mask(shat, float(thr)), g[f"mlp{c}/mask"])
    with pytest.raises(ValueError):
        O.predict_mlp_mask([], 0.0)


def test_importance_filter(golden):
    g = golden("predictor")
    for c in range(8):
        blk, th = g[f"imp{c}/meta"]
        imp = O.block_importance(g[f"imp{c}/z"], int(blk))
        np.testing.assert_array_equal(imp, g[f"imp{c}/imp"])
        np.testing.assert_array_equal(O.filter_neuron_blocks(imp, float(th)), g[f"imp{c}/mask"])


def test_predict_attention_patterns(golden):
    g = golden("predictor")
    for c in range(6):
        nx, n_b = (int(v) for v in g[f"pap{c}/meta"])
        params = O.AttnPredictorParams(list(g[f"pap{c}/wq"]), list(g[f"pap{c}/wk"]))
        xb = [g[f"pap{c}/x{j}"] for j in range(nx)]
        out = O.predict_attention_patterns(xb, params, O.build_pool(n_b), O.PredictorConfig())
        assert out == list(g[f"pap{c}/out"])


# ---------------------------------------------------------------- block-sparse ops
@pytest.mark.parametrize("c", range(5))
def test_block_sparse_ops(golden, c):
    g = golden("block_sparse")
    s, hd, blk = (int(v) for v in g[f"c{c}/meta"])
    n_b = s // blk
    q, k, v, do, coords = (g[f"c{c}/{n}"] for n in ("q", "k", "v", "do", "coords"))
    scale = 1.0 / np.sqrt(hd)
    sc = O.sdd(q, k, coords, blk, scale)
    assert rel(sc, g[f"c{c}/scores"]) < 1e-6
    p = O.sparse_softmax(sc, coords, n_b)
    assert rel(p, g[f"c{c}/probs"]) < 1e-5
    o = O.dsd(p, v, coords, n_b)
    assert rel(o, g[f"c{c}/out"]) < 1e-5
    assert rel(o, g[f"c{c}/dense"]) < 1e-5
    db, dv = O.dsd_backward(p, v, do, coords, n_b)
    assert rel(db, g[f"c{c}/d_blocks"]) < 1e-5 and rel(dv, g[f"c{c}/dv"]) < 1e-5
    ds = O.sparse_softmax_backward(p, db, coords, n_b)
    assert rel(ds, g[f"c{c}/ds"]) < 1e-4
    dq, dk = O.sdd_backward(ds, q, k, coords, blk, scale)
    assert rel(dq, g[f"c{c}/dq"]) < 1e-4 and rel(dk, g[f"c{c}/dk"]) < 1e-4


def test_sparse_softmax_uncovered_row_raises():
    sc = np.zeros((1, 4, 4), np.float32)
    with pytest.raises(O.LayoutError):
        O.sparse_softmax(sc, np.array([[0, 0]]), 2)


# ---------------------------------------------------------------- neuron ops
@pytest.mark.parametrize("c", range(4))
def test_neuron_ops(golden, c):
    g = golden("neuron_ops")
    x, w1, w2, mask = (g[f"c{c}/{n}"] for n in ("x", "w1", "w2", "mask"))
    blk = int(g[f"c{c}/meta"][0])
    h, cols = O.neuron_matmul_fwd1(x, w1, mask, blk)
    np.testing.assert_array_equal(cols, g[f"c{c}/cols"])
    assert rel(h, g[f"c{c}/h"]) < 1e-5 if h.size else g[f"c{c}/h"].size == 0
    out = O.neuron_matmul_fwd2(np.maximum(h, 0), w2, cols)
    assert rel(out, g[f"c{c}/out"]) < 1e-5 if np.abs(g[f"c{c}/out"]).max() > 0 else np.all(out == 0)


def test_active_columns_kat():
    # pkg/tests/test_neuron_ops.py: [T,F,T,F] blk 4 -> [0,1,2,3,8,9,10,11]
    act, cols = O.active_columns(np.array([1, 0, 1, 0], bool), 16, 4)
    assert act == (0, 2) and list(cols) == [0, 1, 2, 3, 8, 9, 10, 11]
    with pytest.raises(O.MaskError):
        O.active_columns(np.ones(3, bool), 16, 4)


# ---------------------------------------------------------------- model / autograd / Adam
@pytest.mark.parametrize("peft", ["lora", "adapter", "bitfit"])
def test_model_step_matches_reference(golden, peft):
    g = golden("model")
    d, H, f, s, L, V, blk, ablk = (int(v) for v in g["dims"])
    dims = O.Dims(d, H, f, s, L, V, blk, ablk)
    m = O.build_model(dims, seed=7, peft=peft)
    assert hashlib.sha256(np.ascontiguousarray(m.layers[1]["w1"].T).tobytes()).hexdigest() == str(g[f"{peft}/hash_w1_l1"])
    assert hashlib.sha256(m.emb.tobytes()).hexdigest() == str(g[f"{peft}/hash_emb"])
    params = O.trainable_params(m)
    for n, p in params.items():
        p[...] = g[f"{peft}/param/{n}"]
    masks = [(list(g[f"{peft}/masks/{i}/heads"]), g[f"{peft}/masks/{i}/neuron"]) for i in range(L)]
    toks = g[f"{peft}/tokens"]
    logits, cache = O.model_forward(m, toks[:-1], masks)
    assert rel(logits, g[f"{peft}/logits"]) < 1e-5
    loss = O.loss_forward(logits, toks[1:])
    assert abs(loss - float(g[f"{peft}/loss"])) < 1e-5
    grads = O.model_backward(m, cache, O.loss_backward(logits, toks[1:]))
    assert set(grads) == set(params)
    for n, gr in grads.items():
        ref = g[f"{peft}/grad/{n}"]
        if np.abs(ref).max() == 0:
            assert np.abs(gr).max() == 0, n
        else:  # bk's true gradient is 0 (softmax shift invariance): absolute floor
            assert np.abs(gr - ref).max() <= 1e-4 * np.abs(ref).max() + 1e-7, n
    # Adam's first step is ~lr*sign(g): feed the reference's own grads so the
    # update itself is checked exactly (sf/autograd.py:203-225)
    O.optimizer_step(params, {}, {}, 0, {n: g[f"{peft}/grad/{n}"] for n in params}, lr=1e-3)
    for n, p in params.items():
        np.testing.assert_array_equal(p, g[f"{peft}/after_adam/{n}"], err_msg=n)


def test_finetune_step_predicted_mode(golden):
    g = golden("finetune_step")
    dims = O.Dims(128, 2, 256, 64, 2, 96, 16, 16)
    m = O.build_model(dims, seed=3, peft="lora")
    attn = [O.AttnPredictorParams(list(g[f"attn{i}/wq"]), list(g[f"attn{i}/wk"])) for i in range(2)]
    mlp = [O.MlpPredictorParams(g[f"mlp{i}/wa"]) for i in range(2)]
    prov = O.PredictedProvider(m, attn, mlp, O.PredictorConfig())
    params = O.trainable_params(m)
    # masks chosen by the predictor must equal the reference's exactly
    for b, seq in enumerate(g["batch"]):
        _, cache = O.model_forward(m, seq[:-1], prov)
        for i, c in enumerate(cache["blocks"]):
            assert c["masks"][0] == list(g["patterns"][b][i])
            np.testing.assert_array_equal(c["masks"][1], g["neuron_masks"][b][i])
    loss, gmean, _ = O.finetune_step(m, g["batch"], prov, params, {}, {}, 0, 1e-3)
    assert abs(loss - float(g["loss"])) < 1e-5
    for n, v in gmean.items():
        ref = g[f"grad/{n}"]
        assert (rel(v, ref) < 1e-4) if np.abs(ref).max() > 0 else np.abs(v).max() == 0, n
    for n, p in params.items():
        assert np.abs(p - g[f"after/{n}"]).max() <= 1e-3 + 1e-7, n  # |update| <= lr; sign of tiny grads may flip


# ---------------------------------------------------------------- exposer oracle mode
def test_exposer_attention(golden):
    """exact_attention -> block_mass -> select_head_pattern / shadowy (sf/exposer.py:47-91,
    sf/harness.py:165-187) against the reference providers' own outputs."""
    g = golden("exposer")
    for c in range(int(g["n_att"])):
        s, n_b, d, H, tau = g[f"att{c}/meta"]
        n_b, H = int(n_b), int(H)
        probs, _ = O.exact_attention(g[f"att{c}/x"], g[f"att{c}/wq"], g[f"att{c}/bq"], g[f"att{c}/wk"],
                                     g[f"att{c}/bk"], H)
        mass = np.stack([O.block_mass(p, n_b) for p in probs])
        np.testing.assert_allclose(mass, g[f"att{c}/mass"], rtol=1e-12, atol=1e-15)
        pool = O.build_pool(n_b)
        assert [O.select_head_pattern(p, pool, float(tau)) for p in probs] == list(g[f"att{c}/pids"])
        assert O.shadowy_pattern(probs, pool, float(tau)) == str(g[f"att{c}/shadowy"][0])


def test_exposer_mlp(golden):
    """OracleProvider._mlp (sf/harness.py:169-176) against the reference."""
    g = golden("exposer")
    for c in range(int(g["n_mlp"])):
        s, d, d_ff, blk, theta, r, scaling = g[f"mlp{c}/meta"]
        a = g.get(f"mlp{c}/a") if int(r) else None
        b = g.get(f"mlp{c}/b") if int(r) else None
        mask, _ = O.oracle_mlp_mask(g[f"mlp{c}/h"], g[f"mlp{c}/w1"], g[f"mlp{c}/b1"], a, b, float(scaling), int(blk),
                                    float(theta))
        np.testing.assert_array_equal(mask, g[f"mlp{c}/mask"])
