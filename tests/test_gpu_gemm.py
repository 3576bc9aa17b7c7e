"""GPU parity of the tcgen05 GEMM engine and the neuron-sparse MLP GEMMs
(K2, sf/neuron_ops.py:75-95, sf/model.py:363-400, sf/autograd.py:97-120)
against a plain PyTorch fp32 reference of the same op. Tolerance: bf16 inputs,
fp32 accumulation -> max|d| / max|ref| <= 1e-2 (bf16 outputs) / 2e-3 (fp32)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _dev():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    return torch.device("cuda")


def rel(a, b):
    a, b = a.float(), b.float()
    return ((a - b).abs().max() / b.abs().max().clamp_min(1e-30)).item()


@pytest.fixture(params=[0, 1, 2, 4, 5], ids=["single_cta", "cta_pair_256", "cta_pair_128", "pair_cluster_mc", "wide_pair"])
def engine(request):
    """All GEMM engine variants: single-CTA tiles, CTA pairs (tcgen05.mma.cta_group::2) with N 256 / 128, and
    clusters of two pairs multicasting the B tile (mode 4)."""
    from paper_2510_15964_b200 import _abi

    prev = _abi.lib().lx_gemm_set_cta_pair(request.param)
    yield request.param
    _abi.lib().lx_gemm_set_cta_pair(prev)


@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (300, 520, 200), (1024, 1024, 1024), (4096, 512, 2048)])
@pytest.mark.parametrize("f32", [True, False])
def test_dense_gemm(M, N, K, f32, engine):
    from paper_2510_15964_b200 import _abi

    dev = _dev()
    g = torch.Generator(device="cpu").manual_seed(M + N + K)
    a = torch.randn(M, K, generator=g).to(dev, torch.bfloat16)
    b = torch.randn(N, K, generator=g).to(dev, torch.bfloat16)
    c = torch.empty(M, N, device=dev, dtype=torch.float32 if f32 else torch.bfloat16)
    _abi.call("lx_gemm_bf16_tn", a.data_ptr(), K, b.data_ptr(), K, c.data_ptr(), N, int(f32), M, N, K, 0, _abi.stream_handle())
    ref = a.float() @ b.float().T
    torch.cuda.synchronize()
    assert rel(c, ref) < (2e-3 if f32 else 1e-2)


def _masks(n_items, n_blk, density, seed):
    rng = np.random.default_rng(seed)
    masks = rng.random((n_items, n_blk)) < density
    if n_items > 1:
        masks[-1] = False  # an empty item
    counts = masks.sum(1).astype(np.int32)
    ids = np.zeros((n_items, n_blk), np.int32)
    for b in range(n_items):
        ids[b, : counts[b]] = np.flatnonzero(masks[b])
    return masks, counts, ids


@pytest.mark.parametrize("n_items,s,d,d_ff,blk,density,r", [(2, 128, 128, 512, 16, 0.5, 8), (3, 100, 192, 384, 16, 0.7, 8),
                                                           (4, 512, 2048, 8192, 16, 0.2, 8), (2, 256, 256, 1024, 32, 0.4, 0),
                                                           (2, 128, 128, 512, 64, 0.6, 4)])
@pytest.mark.parametrize("packed", [False, True])
def test_neuron_mlp_gemms(n_items, s, d, d_ff, blk, density, r, packed, engine):
    from paper_2510_15964_b200 import _abi

    dev = _dev()
    st = _abi.stream_handle()
    n_blk = d_ff // blk
    masks, counts, ids = _masks(n_items, n_blk, density, seed=d + d_ff)
    g = torch.Generator(device="cpu").manual_seed(7)
    M = n_items * s
    x = (torch.randn(M, d, generator=g)).to(dev, torch.bfloat16)
    w1t = (torch.randn(d_ff, d, generator=g) * d ** -0.5).to(dev, torch.bfloat16)
    w2 = (torch.randn(d_ff, d, generator=g) * d_ff ** -0.5).to(dev, torch.bfloat16)
    b1 = torch.randn(d_ff, generator=g).to(dev) * 0.1
    b2 = torch.randn(d, generator=g).to(dev) * 0.1
    rr = max(r, 1)
    ax1 = torch.randn(M, rr, generator=g).to(dev)
    B1 = torch.randn(rr, d_ff, generator=g).to(dev) * 0.1
    ax2 = torch.randn(M, rr, generator=g).to(dev)
    B2 = torch.randn(rr, d, generator=g).to(dev) * 0.1
    A1 = torch.randn(d, rr, generator=g).to(dev) * 0.1
    A2 = torch.randn(d_ff, rr, generator=g).to(dev) * 0.1
    dax1 = torch.randn(M, rr, generator=g).to(dev)
    dax2 = torch.randn(M, rr, generator=g).to(dev)
    d_out = torch.randn(M, d, generator=g).to(dev, torch.bfloat16)
    cnt_d = torch.from_numpy(counts).to(dev)
    ids_d = torch.from_numpy(ids).to(dev)
    ld_h = d_ff
    scaling = 0.5
    a = torch.zeros(M, ld_h, device=dev, dtype=torch.bfloat16)
    P = lambda t: None if (t is None or r == 0) else t.data_ptr()  # noqa: E731
    WP1 = WP2 = None
    if packed:  # item-packed active rows (lx_pack_active_rows) -> kPackedN / kPackedK GEMMs
        w1p = torch.empty(n_items, d_ff, d, device=dev, dtype=torch.bfloat16)
        w2p = torch.empty(n_items, d_ff, d, device=dev, dtype=torch.bfloat16)
        for src, dst in ((w1t, w1p), (w2, w2p)):
            _abi.call("lx_pack_active_rows", src.data_ptr(), d_ff, d, blk, n_items, cnt_d.data_ptr(), ids_d.data_ptr(),
                      dst.data_ptr(), st)
        WP1, WP2 = w1p.data_ptr(), w2p.data_ptr()
    bits = torch.zeros(M, ld_h // 16, device=dev, dtype=torch.int16) if ld_h % 16 == 0 else None
    _abi.call("lx_neuron_fc1", x.data_ptr(), n_items, s, d, d_ff, blk, w1t.data_ptr(), cnt_d.data_ptr(), ids_d.data_ptr(),
              b1.data_ptr(), P(ax1), P(B1), r, scaling, 1, a.data_ptr(), ld_h, WP1, _abi.ptr(bits), st)
    out = torch.empty(M, d, device=dev, dtype=torch.bfloat16)
    _abi.call("lx_neuron_fc2", a.data_ptr(), ld_h, n_items, s, d, d_ff, blk, w2.data_ptr(), cnt_d.data_ptr(), ids_d.data_ptr(),
              b2.data_ptr(), P(ax2), P(B2), r, scaling, out.data_ptr(), 0, None, WP2, st)
    dz = torch.zeros(M, ld_h, device=dev, dtype=torch.bfloat16)
    _abi.call("lx_neuron_fc2_dgrad", d_out.data_ptr(), n_items, s, d, d_ff, blk, w2.data_ptr(), cnt_d.data_ptr(),
              ids_d.data_ptr(), P(dax2), P(A2), r, a.data_ptr(), dz.data_ptr(), ld_h, WP2, None, st)
    if bits is not None:  # relu'(z) from fc1's bits instead of the bf16 activation: the same dz bits
        dz_b = torch.zeros_like(dz)
        _abi.call("lx_neuron_fc2_dgrad", d_out.data_ptr(), n_items, s, d, d_ff, blk, w2.data_ptr(), cnt_d.data_ptr(),
                  ids_d.data_ptr(), P(dax2), P(A2), r, a.data_ptr(), dz_b.data_ptr(), ld_h, WP2, bits.data_ptr(), st)
        torch.cuda.synchronize()
        assert torch.equal(dz_b, dz)
    dx = torch.empty(M, d, device=dev, dtype=torch.bfloat16)
    _abi.call("lx_neuron_fc1_dgrad", dz.data_ptr(), ld_h, n_items, s, d, d_ff, blk, w1t.data_ptr(), cnt_d.data_ptr(),
              ids_d.data_ptr(), P(dax1), P(A1), r, dx.data_ptr(), 0, WP1, st)
    torch.cuda.synchronize()
    for b in range(n_items):
        rows = slice(b * s, (b + 1) * s)
        cols = torch.from_numpy((ids[b, : counts[b], None] * blk + np.arange(blk)[None]).reshape(-1)).to(dev)
        F = cols.numel()
        xb = x[rows].float()
        z = xb @ w1t[cols].float().T + b1[cols]
        if r:
            z = z + scaling * ax1[rows] @ B1[:, cols]
        aref = torch.relu(z)
        if F:
            assert rel(a[rows, :F], aref) < 1e-2
        ab = a[rows, :F].float()  # chain on the GPU's own bf16 hidden
        o = ab @ w2[cols].float() + b2
        if r:
            o = o + scaling * ax2[rows] @ B2
        assert rel(out[rows], o) < 1e-2
        da = d_out[rows].float() @ w2[cols].float().T
        if r:
            da = da + dax2[rows] @ A2[cols].T
        dzr = da * (ab > 0)
        if F:
            assert rel(dz[rows, :F], dzr) < 1e-2
        dxr = dz[rows, :F].float() @ w1t[cols].float()
        if r:
            dxr = dxr + dax1[rows] @ A1.T
        assert rel(dx[rows], dxr) < 1e-2 if dxr.abs().max() > 0 else dx[rows].float().abs().max() == 0


@pytest.mark.parametrize("gather", [False, True])
@pytest.mark.parametrize("r,w_layout", [(8, "kr"), (8, "rk"), (16, "kr"), (12, "rk"), (4, "rk"), (1, "kr")])
def test_lora_skinny_kernels(gather, r, w_layout):
    """rowproj / colgrad (csrc/lora.cu) vs torch fp32 on the same bf16 operands, incl. per-item gathers."""
    from paper_2510_15964_b200 import neuron_ops as N

    dev = _dev()
    n_items, s, K, blk = 3, 300, 1024, 16
    n_blk = K // blk
    masks, counts, ids = _masks(n_items, n_blk, 0.4, seed=r)
    g = torch.Generator(device="cpu").manual_seed(r)
    x = torch.randn(n_items * s, K, generator=g).to(dev, torch.bfloat16)
    w = (torch.randn(K, r, generator=g) if w_layout == "kr" else torch.randn(r, K, generator=g)).to(dev)
    w_sk, w_sq = (r, 1) if w_layout == "kr" else (1, K)
    wk = w if w_layout == "kr" else w.t()
    nm = N.lower_mask(torch.from_numpy(masks).to(dev), n_blk, blk, n_items, dev) if gather else None
    y = N.rowproj(x, n_items, s, K, w, w_sk, w_sq, r, scale=0.5, masks=nm, blk=blk)
    p = torch.randn(n_items * s, r, generator=g).to(dev)
    G = torch.empty(r, K, device=dev)
    N.colgrad(p, x, n_items, s, K, r, 0.25, G, K, 1, masks=nm, blk=blk)
    torch.cuda.synchronize()
    Gref = torch.zeros(r, K, device=dev)
    for b in range(n_items):
        rows = slice(b * s, (b + 1) * s)
        if gather:
            cols = torch.from_numpy((ids[b, : counts[b], None] * blk + np.arange(blk)[None]).reshape(-1)).to(dev)
            xb = x[rows, : cols.numel()].float()  # packed columns
            yr = 0.5 * xb @ wk[cols]
            Gref[:, cols] += 0.25 * p[rows].t() @ xb
        else:
            yr = 0.5 * x[rows].float() @ wk
            Gref += 0.25 * p[rows].t() @ x[rows].float()
        assert rel(y[rows], yr) < 1e-4 if yr.abs().max() > 0 else y[rows].abs().max() == 0
    assert rel(G, Gref) < 1e-4
    if gather:  # inactive columns exactly zero
        act = np.zeros(K, bool)
        for b in range(n_items):
            act[(ids[b, : counts[b], None] * blk + np.arange(blk)[None]).reshape(-1)] = True
        assert float(G[:, torch.from_numpy(~act).to(dev)].abs().max()) == 0


@pytest.mark.parametrize("M,N,K,r,mode", [(4096, 6144, 2048, 16, "bf16"), (300, 520, 200, 8, "f32"), (512, 2048, 2048, 8, "resid"),
                                          (256, 256, 64, 0, "bf16"), (4096, 2048, 2112, 0, "bf16"), (1000, 1000, 320, 3, "f32")])
@pytest.mark.parametrize("kn", [False, True], ids=["b_nk", "b_kn"])
def test_linear_fused_epilogue(M, N, K, r, mode, kn, engine):
    """lx_linear / lx_linear_kn: out = (resid) + A B^T + bias + s * lora_x . w (lora_linear_forward's fused
    dense product), weight K-major [N, K] or as stored for x @ W ([K, N], the projections' layout)."""
    from paper_2510_15964_b200 import model as Mo

    dev = _dev()
    g = torch.Generator(device="cpu").manual_seed(M + r)
    a = torch.randn(M, K, generator=g).to(dev, torch.bfloat16)
    bt = (torch.randn(N, K, generator=g) * K ** -0.5).to(dev, torch.bfloat16)
    bias = torch.randn(N, generator=g).to(dev)
    lx = torch.randn(M, max(r, 1), generator=g).to(dev)
    lw = torch.randn(max(r, 1), N, generator=g).to(dev) * 0.1
    resid = torch.randn(M, N, generator=g).to(dev) if mode == "resid" else None
    w = bt.t().contiguous() if kn else bt
    if kn and N % 8:
        pytest.skip("[K, N] weight rows need N % 8 == 0 (16-byte TMA row stride)")
    out = Mo.linear(a, w, out_f32=mode != "bf16", resid=resid, bias=bias, lora_x=lx if r else None, lora_w=lw if r else None,
                    w_sr=N, w_sc=1, r=r, scaling=0.5, kn=kn)
    ref = a.float() @ bt.float().T + bias
    if r:
        ref = ref + 0.5 * lx @ lw
    if resid is not None:
        ref = ref + resid
    torch.cuda.synchronize()
    assert out.dtype == (torch.bfloat16 if mode == "bf16" else torch.float32)
    assert rel(out, ref) < (1e-2 if mode == "bf16" else 2e-3)


def test_cross_entropy_kernel():
    """Fused LM-head CE fwd+bwd (csrc/ce.cu) vs torch fp32 (sf/model.py:454-472)."""
    from paper_2510_15964_b200.engine import lm_head_loss_and_grad

    dev = _dev()
    g = torch.Generator(device="cpu").manual_seed(3)
    B, s, d, V = 2, 96, 128, 1000
    hf = torch.randn(B * s, d, generator=g).to(dev, torch.bfloat16)
    emb = (torch.randn(V, d, generator=g) * 0.3).to(dev, torch.bfloat16)
    tgt = torch.randint(0, V, (B * s,), generator=g).to(dev)
    loss, d_hf = lm_head_loss_and_grad(hf, emb, tgt, s, chunk=64)
    logits = (hf.float() @ emb.float().T).requires_grad_(True)
    ref = torch.nn.functional.cross_entropy(logits, tgt)
    (ref * B).backward()  # per-item mean summed over items == gradient convention of loss_backward (1/s)
    ref_dhf = logits.grad @ emb.float()
    torch.cuda.synchronize()
    assert abs(float(loss) - float(ref)) < 1e-4 * float(ref)
    assert rel(d_hf, ref_dhf) < 1e-2


@pytest.mark.parametrize("rows,d,V,scale", [(192, 128, 1000, 0.3), (700, 768, 50272, 0.05), (4096, 2048, 50272, 0.03),
                                          (300, 256, 517, 2.0)])
def test_lm_head_fused_ce(rows, d, V, scale):
    """lx_lm_head_ce (logits GEMM with the CE epilogue, combine, rescale) vs float64 torch (sf/model.py:449-472):
    per-row losses at 1e-5 relative (fp32 statistics), the bf16 gradient g = (softmax - onehot) / s at 1e-2 with
    the one-hot on the target column only, and d_hf = g emb through the engine's helper at 1e-2. Ragged V
    (not a multiple of the 512-column tile or of 8), targets on the first and last columns, wide logits."""
    from paper_2510_15964_b200 import _abi
    from paper_2510_15964_b200.engine import lm_head_loss_and_grad

    dev = _dev()
    g0 = torch.Generator(device="cpu").manual_seed(rows + V)
    hf = torch.randn(rows, d, generator=g0).to(dev, torch.bfloat16)
    emb = (torch.randn(V, d, generator=g0) * scale).to(dev, torch.bfloat16)
    tgt = torch.randint(0, V, (rows,), generator=g0).to(dev)
    tgt[0], tgt[1] = 0, V - 1
    s = 37
    nseg = _abi.lib().lx_lm_head_ce_nseg(V)
    ldg = (V + 7) // 8 * 8
    gbuf = torch.empty(rows, ldg, dtype=torch.bfloat16, device=dev)
    stats = torch.empty(rows, 2 * nseg, device=dev)
    coef = torch.empty(rows, nseg, device=dev)
    tl = torch.empty(rows, device=dev)
    row_loss = torch.empty(rows, device=dev)
    _abi.call("lx_lm_head_ce", hf.data_ptr(), d, rows, d, emb.data_ptr(), V, tgt.data_ptr(), 1.0 / s, gbuf.data_ptr(), ldg,
              stats.data_ptr(), coef.data_ptr(), tl.data_ptr(), row_loss.data_ptr(), _abi.stream_handle(dev))
    torch.cuda.synchronize()
    logits = hf.double() @ emb.double().T
    ref_loss = torch.nn.functional.cross_entropy(logits, tgt, reduction="none")
    ref_g = (torch.softmax(logits, dim=1) - torch.nn.functional.one_hot(tgt, V).double()) / s
    assert (row_loss.double() - ref_loss).abs().max().item() < 1e-5 * ref_loss.abs().max().item()
    gv = gbuf[:, :V]
    assert rel(gv.float(), ref_g) < 1e-2
    assert torch.equal(gv[:, 0].float() < 0, tgt == 0)
    loss, d_hf = lm_head_loss_and_grad(hf, emb, tgt, s)
    torch.cuda.synchronize()
    assert abs(float(loss) - float(ref_loss.mean())) < 1e-5 * float(ref_loss.mean())
    assert rel(d_hf, ref_g @ emb.double()) < 1e-2


def test_cross_entropy_kernel_persistent_rows():
    """More rows than the persistent CE grid (2 CTAs per SM) at the OPT vocabulary (V % 1024 != 0):
    every row's loss and gradient vs torch fp32, so rows handled on a CTA's second and later passes
    are covered (sf/model.py:454-472)."""
    from paper_2510_15964_b200 import _abi

    dev = _dev()
    g = torch.Generator(device="cpu").manual_seed(5)
    rows, V = 2 * torch.cuda.get_device_properties(0).multi_processor_count + 77, 50272
    logits = (torch.randn(rows, V, generator=g) * 3).to(dev)
    tgt = torch.randint(0, V, (rows,), generator=g).to(dev)
    tgt[0], tgt[1] = 0, V - 1  # first and last column as targets
    row_loss = torch.empty(rows, dtype=torch.float32, device=dev)
    gb = torch.empty(rows, V, dtype=torch.bfloat16, device=dev)
    inv_s = 1.0 / 37
    _abi.call("lx_cross_entropy", logits.data_ptr(), rows, V, tgt.data_ptr(), inv_s, row_loss.data_ptr(), gb.data_ptr(),
              _abi.stream_handle(logits.device))
    torch.cuda.synchronize()
    ref_loss = torch.nn.functional.cross_entropy(logits, tgt, reduction="none")
    ref_g = (torch.softmax(logits, dim=1) - torch.nn.functional.one_hot(tgt, V).float()) * inv_s
    assert (row_loss - ref_loss).abs().max().item() < 1e-4 * ref_loss.abs().max().item()
    assert rel(gb.float(), ref_g) < 1e-2
    assert torch.equal(gb[:, 0].float() < 0, tgt == 0)  # the one-hot lands on the target column only


@pytest.mark.parametrize("gather", [False, True])
@pytest.mark.parametrize("r,rp", [(8, 8), (16, 16), (4, 8), (12, 16)])
@pytest.mark.parametrize("K", [1024, 4096])
def test_rowproj_packed_and_pack_params(gather, r, rp, K):
    """lx_pack_params (fp32 LoRA factor -> bf16 hi/lo pack) feeding lx_rowproj_packed, dense and gathered
    through the item's active block ids, with the optional bf16 copy of Y (K-extended GEMM columns). K 1024:
    32-row CTAs with a ragged last CTA; K 4096: the 16-row variant."""
    from paper_2510_15964_b200 import _abi, neuron_ops as N

    dev = _dev()
    n_items, s, blk = 3, 300, 16
    n_blk = K // blk
    masks, counts, ids = _masks(n_items, n_blk, 0.4, seed=r + rp)
    g = torch.Generator(device="cpu").manual_seed(r)
    x = torch.randn(n_items * s, K + 16, generator=g).to(dev, torch.bfloat16)[:, :K]  # row stride K + 16
    a = torch.randn(K, r, generator=g).to(dev)  # W(k, q) = A[k][q]
    wp = torch.zeros(2, rp, K, dtype=torch.bfloat16, device=dev)
    seg = _abi.PackSegment(a.data_ptr(), 1, r, r, K, wp.data_ptr(), K, 1, rp * K, 1.0, 0)
    segs = torch.frombuffer(bytearray(bytes(seg)), dtype=torch.uint8).to(dev)
    _abi.call("lx_pack_params", segs.data_ptr(), 1, _abi.stream_handle())
    torch.cuda.synchronize()
    assert rel(wp[0, :r].float() + wp[1, :r].float(), a.t()) < 1e-5  # hi + lo keeps ~16 mantissa bits
    nm = N.lower_mask(torch.from_numpy(masks).to(dev), n_blk, blk, n_items, dev) if gather else None
    yb = torch.zeros(n_items * s, 24, dtype=torch.bfloat16, device=dev)
    y = N.rowproj_packed(x, n_items, s, K, wp, r, scale=0.5, masks=nm, blk=blk, out_bf16=yb[:, 3 : 3 + r])
    torch.cuda.synchronize()
    for b in range(n_items):
        rows = slice(b * s, (b + 1) * s)
        if gather:
            cols = torch.from_numpy((ids[b, : counts[b], None] * blk + np.arange(blk)[None]).reshape(-1)).to(dev)
            ref = 0.5 * x[rows, : cols.numel()].float() @ a[cols]
        else:
            ref = 0.5 * x[rows].float() @ a
        assert rel(y[rows], ref) < 1e-4 if ref.abs().max() > 0 else y[rows].abs().max() == 0
        assert rel(yb[rows, 3 : 3 + r], ref) < 1e-2 if ref.abs().max() > 0 else True
    assert yb[:, :3].abs().max() == 0 and yb[:, 3 + r :].abs().max() == 0  # only the r columns are written


def test_colgrad_group_mixed_problems():
    """One lx_colgrad_group launch over dense, gathered (packed per-item columns), column-sum and
    rank-16 problems with strided X / P / G — each equal to its own torch fp32 reduction."""
    from paper_2510_15964_b200 import neuron_ops as N

    dev = _dev()
    n_items, s, d, f, blk = 4, 320, 512, 2048, 16
    n_blk = f // blk
    masks, counts, ids = _masks(n_items, n_blk, 0.3, seed=5)
    nm = N.lower_mask(torch.from_numpy(masks).to(dev), n_blk, blk, n_items, dev)
    g = torch.Generator(device="cpu").manual_seed(11)
    M = n_items * s
    xw = torch.randn(M, 3 * d + 16, generator=g).to(dev, torch.bfloat16)  # dense X: a column slice, row stride 3d+16
    xd = xw[:, d : 2 * d]
    fa = int(counts.max()) * blk
    xp = torch.randn(M, fa + 8, generator=g).to(dev, torch.bfloat16)  # packed X
    p16 = torch.randn(M, 24, generator=g).to(dev)
    g1 = torch.empty(8, d, device=dev)          # G(q, c) = g[q*d + c]
    g2 = torch.empty(f, 8, device=dev)          # transposed: G(q, c) = g[c*8 + q]
    g3 = torch.empty(d, device=dev)             # column sums
    g4 = torch.empty(16, d, device=dev)         # rank 16
    probs = [N.colgrad_problem(p16[:, :8], xd, d, 8, 0.5, g1, d, 1),
             N.colgrad_problem(p16[:, 8:16], xp, f, 8, 1.0, g2, 1, 8, masks=nm, blk=blk),
             N.colgrad_problem(None, xd, d, 1, 1.0, g3, 0, 1),
             N.colgrad_problem(p16[:, 4:20], xd, d, 16, 2.0, g4, d, 1)]
    N.colgrad_group(probs, n_items, s)
    torch.cuda.synchronize()
    assert rel(g1, 0.5 * p16[:, :8].t() @ xd.float()) < 1e-4
    ref2 = torch.zeros(8, f, device=dev)
    for b in range(n_items):
        rows = slice(b * s, (b + 1) * s)
        cols = torch.from_numpy((ids[b, : counts[b], None] * blk + np.arange(blk)[None]).reshape(-1)).to(dev)
        ref2[:, cols] += p16[rows, 8:16].t() @ xp[rows, : cols.numel()].float()
    assert rel(g2.t(), ref2) < 1e-4
    act = np.zeros(f, bool)
    for b in range(n_items):
        act[(ids[b, : counts[b], None] * blk + np.arange(blk)[None]).reshape(-1)] = True
    assert float(g2[torch.from_numpy(~act).to(dev)].abs().max()) == 0  # inactive columns exactly 0
    assert rel(g3, xd.float().sum(0)) < 1e-4
    assert rel(g4, 2.0 * p16[:, 4:20].t() @ xd.float()) < 1e-4
    # deterministic: a second launch gives identical bits
    g1b = g1.clone()
    N.colgrad_group(probs, n_items, s)
    torch.cuda.synchronize()
    assert torch.equal(g1, g1b)


def test_adam_step_kernel():
    """lx_adam_step (one pass, float64 moments) vs the reference update order of sf/autograd.py:218-224
    evaluated in float64 with NumPy, over three steps."""
    from paper_2510_15964_b200 import _abi

    dev = _dev()
    rng = np.random.default_rng(4)
    n = 100003
    p0 = rng.standard_normal(n).astype(np.float32) * 0.02
    p = torch.from_numpy(p0.copy()).to(dev)
    m = torch.zeros(n, dtype=torch.float64, device=dev)
    v = torch.zeros(n, dtype=torch.float64, device=dev)
    pr, mr, vr = p0.copy(), np.zeros(n), np.zeros(n)
    lr, b1, b2, eps = 1e-3, 0.9, 0.999, 1e-8
    for t in range(1, 4):
        g = rng.standard_normal(n).astype(np.float32) * 1e-3
        _abi.call("lx_adam_step", p.data_ptr(), torch.from_numpy(g).to(dev).data_ptr(), m.data_ptr(), v.data_ptr(), n, lr,
                  b1, b2, eps, t, _abi.stream_handle())
        torch.cuda.synchronize()
        gd = g.astype(np.float64)
        mr = b1 * mr + (1 - b1) * gd
        vr = b2 * vr + (1 - b2) * gd * gd
        pr -= (lr * (mr / (1 - b1**t)) / (np.sqrt(vr / (1 - b2**t)) + eps)).astype(np.float32)
    assert np.abs(m.cpu().numpy() - mr).max() <= 1e-15
    assert np.abs(v.cpu().numpy() - vr).max() <= 1e-15
    assert np.abs(p.cpu().numpy() - pr).max() <= 1e-7


@pytest.mark.parametrize("d", [768, 1024, 2048, 4096, 5120])
@pytest.mark.parametrize("with_delta", [False, True])
def test_layernorm_fwd_kernel(d, with_delta):
    """lx_layernorm_fwd (csrc/layernorm.cu) vs torch fp32 (sf/model.py:307-312): fused residual add
    (bit-exact fp32 sum), mean / inv-std, bf16 output and the fused downsampled rows
    (sf/predictor.py:62-71). M spans several row passes of the persistent grid with a ragged last pass."""
    from paper_2510_15964_b200 import _abi

    dev = _dev()
    g = torch.Generator(device="cpu").manual_seed(11)
    n_items, s, m_small = 7, 700, 26  # M = 4900 rows
    M = n_items * s
    x = torch.randn(M, d, generator=g).to(dev)
    delta = torch.randn(M, d, generator=g).to(dev, torch.bfloat16) if with_delta else None
    gamma = (1 + 0.1 * torch.randn(d, generator=g)).to(dev)
    beta = (0.1 * torch.randn(d, generator=g)).to(dev)
    resid = torch.empty(M, d, device=dev) if with_delta else None
    y = torch.empty(M, d, dtype=torch.bfloat16, device=dev)
    mean = torch.empty(M, device=dev)
    istd = torch.empty(M, device=dev)
    xs = torch.zeros(n_items * m_small, d, dtype=torch.bfloat16, device=dev)
    _abi.call("lx_layernorm_fwd", x.data_ptr(), _abi.ptr(delta), _abi.ptr(resid), M, d, gamma.data_ptr(), beta.data_ptr(),
              1e-5, y.data_ptr(), d, mean.data_ptr(), istd.data_ptr(), s, m_small, xs.data_ptr(), _abi.stream_handle(dev))
    torch.cuda.synchronize()
    h = x + delta.float() if with_delta else x
    if with_delta:
        assert torch.equal(resid, h)
    ref = torch.nn.functional.layer_norm(h, (d,), gamma, beta, 1e-5)
    assert rel(y.float(), ref) < 1e-2
    assert torch.allclose(mean, h.mean(1), atol=1e-5)
    assert torch.allclose(istd, 1 / torch.sqrt(h.var(1, unbiased=False) + 1e-5), rtol=1e-4)
    idx = torch.tensor([(i * s) // m_small for i in range(m_small)], device=dev)
    want = y.view(n_items, s, d)[:, idx].reshape(-1, d)
    assert torch.equal(xs, want)


@pytest.mark.parametrize("d", [768, 2048, 4096, 5120])
@pytest.mark.parametrize("dy_f32", [False, True])
def test_layernorm_bwd_kernel(d, dy_f32):
    """lx_layernorm_bwd (warp kernel up to d = 2048, block kernel above): dx_accum += LN'(dy) against torch autograd
    of layer_norm in float64, and the bf16 copy of the updated accumulator."""
    from paper_2510_15964_b200 import _abi

    dev = _dev()
    g = torch.Generator(device="cpu").manual_seed(d)
    M = 1000
    x = torch.randn(M, d, generator=g).to(dev)
    gamma = (1 + 0.1 * torch.randn(d, generator=g)).to(dev)
    beta = torch.zeros(d, device=dev)
    dy = torch.randn(M, d, generator=g).to(dev)
    dy_in = dy if dy_f32 else dy.to(torch.bfloat16)
    acc0 = torch.randn(M, d, generator=g).to(dev)
    acc = acc0.clone()
    y = torch.empty(M, d, dtype=torch.bfloat16, device=dev)
    mean, istd = torch.empty(M, device=dev), torch.empty(M, device=dev)
    st = _abi.stream_handle(dev)
    _abi.call("lx_layernorm_fwd", x.data_ptr(), None, None, M, d, gamma.data_ptr(), beta.data_ptr(), 1e-5, y.data_ptr(), d,
              mean.data_ptr(), istd.data_ptr(), 0, 0, None, st)
    ob = torch.empty(M, d, dtype=torch.bfloat16, device=dev)
    _abi.call("lx_layernorm_bwd", dy_in.data_ptr(), int(dy_f32), x.data_ptr(), gamma.data_ptr(), mean.data_ptr(),
              istd.data_ptr(), M, d, acc.data_ptr(), ob.data_ptr(), st)
    torch.cuda.synchronize()
    xd = x.double().requires_grad_(True)
    out = torch.nn.functional.layer_norm(xd, (d,), gamma.double(), beta.double(), 1e-5)
    out.backward(dy_in.double())
    ref = acc0.double() + xd.grad
    assert rel(acc, ref) < 1e-4
    assert torch.equal(ob, acc.to(torch.bfloat16))


def test_rowproj_packed_seg_matches_per_segment():
    """lx_rowproj_packed_seg (q/k/v LoRA input-grad projections in one launch) gives the bits of one
    lx_rowproj_packed call per segment, on strided column slices of a fused [M, 3d + kx] operand."""
    from paper_2510_15964_b200 import neuron_ops as N

    dev = _dev()
    M_, d, r, n_t = 1000, 512, 8, 2
    g = torch.Generator().manual_seed(11)
    xfull = (torch.randn(M_, 3 * d + 16, generator=g) * 0.5).to(dev, torch.bfloat16)
    packs = (torch.randn(n_t, 2, 8, d, generator=g) * 0.1).to(dev, torch.bfloat16)
    slots = [0, 2]
    y = torch.full((M_, n_t * r), float("nan"), device=dev)
    yb = torch.full((M_, 3 * d + 16), 7.0, dtype=torch.bfloat16, device=dev)
    N.rowproj_packed_seg(xfull[:, slots[0] * d:], (slots[1] - slots[0]) * d, d, packs, r, 0.5, y, r, yb[:, 3 * d:], r, n_t)
    ref = torch.empty(M_, n_t * r, device=dev)
    refb = torch.full_like(yb, 7.0)
    for j, sl in enumerate(slots):
        N.rowproj_packed(xfull[:, sl * d:(sl + 1) * d], 1, M_, d, packs[j], r, scale=0.5, out=ref[:, j * r:(j + 1) * r],
                         out_bf16=refb[:, 3 * d + j * r:3 * d + (j + 1) * r])
    torch.cuda.synchronize()
    assert torch.equal(y, ref)
    assert torch.equal(yb, refb)
