#!/usr/bin/env python
"""Operator sweep, BASELINE.json configs[1]: the isolated sparse operators at OPT-1.3B layer
shapes (d 2048, H 32, hd 64, d_ff 8192, s 1024, B 4 -> M 4096 tokens) on 1 B200, 50-90%
sparsity, reported as effective TFLOP/s on ACTIVE FLOPs next to (a) the same kernels with a
full mask / dense layout (the reference bench's own baseline, sf/bench.py:64-117) and (b) the
dense cuBLAS / SDPA bf16 op of the same shape.

    python bench_ops.py [--reps 20] [--ops mlp,attn] [--sparsity 0.5,0.75,0.9]

One JSON line per (op, phase, sparsity). Masks follow the reference bench: neuron masks are
`_spread_mask` (evenly spread active blocks, sf/bench.py:45-51), attention layouts
`_attn_layout` (diagonal kept, seeded random off-diagonal, sf/bench.py:54-62), one layout per
head. Every launch is timed alone with CUDA events on the launching stream after an L2 flush
(a 512 MB write), median over reps.

Active FLOPs: MLP fwd = 2 GEMMs x 2*M*d*F_act, MLP bwd (input grads, frozen
weights) = 2 x 2*M*d*F_act; attention fwd = 4*B*H*nnz*blk^2*hd, bwd = 8*B*H*nnz*blk^2*hd
(reference MAC convention sf/block_sparse.py:58-59,124-125; the flash recompute of QK^T is
not credited).
"""

from __future__ import annotations

import argparse
import json
import statistics
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CFG2 = dict(d=2048, H=32, hd=64, d_ff=8192, s=1024, B=4, blk=16)


def spread_mask(n_blk: int, sparsity: float) -> np.ndarray:
    """sf/bench.py:45-51."""
    n_active = max(1, round((1.0 - sparsity) * n_blk))
    idx = np.unique((np.arange(n_active) * n_blk) // n_active)
    m = np.zeros(n_blk, dtype=bool)
    m[idx] = True
    return m


def attn_layout(n_b: int, sparsity: float, rng) -> list[tuple[int, int]]:
    """sf/bench.py:54-62 (seeded PCG64 like sf/tensor_core.py:19-21)."""
    coords = {(i, i) for i in range(n_b)}
    want = max(n_b, round((1.0 - sparsity) * n_b * n_b))
    off = [(i, j) for i in range(n_b) for j in range(n_b) if i != j]
    rng.shuffle(off)
    for c in off[: max(0, want - n_b)]:
        coords.add(c)
    return sorted(coords)


class Timer:
    """Median device time of fn() over reps, each launch after an L2 flush, events on the current stream."""

    def __init__(self):
        import torch

        self.flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")

    def __call__(self, fn, reps: int, warmup: int = 3) -> float:
        import torch

        for _ in range(warmup):
            fn()
        ts = []
        for _ in range(reps):
            self.flush.fill_(1)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            b.synchronize()
            ts.append(a.elapsed_time(b))
        return statistics.median(ts)


def line(op, phase, sp, ms, flops, peak, extra=None):
    tf = flops / (ms * 1e-3) / 1e12
    out = {"op": op, "phase": phase, "sparsity": sp, "ms": round(ms, 4), "active_gflop": round(flops / 1e9, 2),
           "eff_tflops": round(tf, 1), "frac_of_peak": round(tf / peak, 3)}
    out.update(extra or {})
    print(json.dumps(out), flush=True)
    return out


def sweep_mlp(args, timer, peak):
    import torch

    from paper_2510_15964_b200 import neuron_ops as N

    c = CFG2
    d, f, blk, B, s = c["d"], c["d_ff"], c["blk"], c["B"], c["s"]
    M = B * s
    g = torch.Generator(device="cuda").manual_seed(0)
    x = (torch.randn(M, d, device="cuda", generator=g)).to(torch.bfloat16)
    dO = (torch.randn(M, d, device="cuda", generator=g) * 0.1).to(torch.bfloat16)
    w1 = (torch.randn(d, f, device="cuda", generator=g) * 0.02)
    w2 = (torch.randn(f, d, device="cuda", generator=g) * 0.02)
    lw = N.LayeredWeights.from_row_major(w1, w2, "cuda")
    b1 = torch.zeros(f, device="cuda")
    n_blk = f // blk
    rows = []
    dense_ms = {}
    for sp in [0.0] + args.sparsity:
        mask = spread_mask(n_blk, sp)
        nm = N.lower_mask(mask, n_blk, blk, B, "cuda")
        f_act = int(mask.sum()) * blk
        hid_buf = torch.empty(M, f, dtype=torch.bfloat16, device="cuda")
        out = torch.empty(M, d, dtype=torch.bfloat16, device="cuda")
        state = {}

        def fwd():
            w1p = N.pack_active_rows(lw.w1_t, nm)
            w2p = N.pack_active_rows(lw.w2, nm)
            hid = N.neuron_matmul_fwd1(x.view(B, s, d), lw, nm, blk, bias=b1, relu=True, out=hid_buf, w_packed=w1p)
            N.neuron_matmul_fwd2(hid, lw, None, out=out, w_packed=w2p)
            state.update(w1p=w1p, w2p=w2p, hid=hid)

        fwd()
        from paper_2510_15964_b200 import _abi

        dz = torch.empty(M, f, dtype=torch.bfloat16, device="cuda")
        dx = torch.empty(M, d, dtype=torch.bfloat16, device="cuda")
        st = _abi.stream_handle(x.device)

        def bwd():
            a = state["hid"].values
            _abi.call("lx_neuron_fc2_dgrad", dO.data_ptr(), B, s, d, f, blk, lw.w2.data_ptr(), nm.counts.data_ptr(),
                      nm.ids.data_ptr(), 0, 0, 0, a.data_ptr(), dz.data_ptr(), a.stride(0), state["w2p"].data_ptr(), None,
                      st)
            _abi.call("lx_neuron_fc1_dgrad", dz.data_ptr(), dz.stride(0), B, s, d, f, blk, lw.w1_t.data_ptr(),
                      nm.counts.data_ptr(), nm.ids.data_ptr(), 0, 0, 0, dx.data_ptr(), 0, state["w1p"].data_ptr(), st)

        fl = 2 * 2.0 * M * d * f_act
        for phase, fn in (("fwd", fwd), ("bwd", bwd)):
            ms = timer(fn, args.reps)
            if sp == 0.0:
                dense_ms[phase] = ms
            rows.append(line("neuron_mlp", phase, sp, ms, fl, peak, {
                "active_blocks": int(mask.sum()), "n_blk": n_blk, "M": M, "d": d, "d_ff": f,
                "speedup_vs_same_kernel_dense": round(dense_ms[phase] / ms, 3),
                "kernels": "pack_rows x2 + fc1(+b1,ReLU) + fc2" if phase == "fwd" else "fc2_dgrad(relu') + fc1_dgrad"}))
    # dense cuBLAS of the same op
    w1b, w2b = w1.to(torch.bfloat16), w2.to(torch.bfloat16)

    def dfwd():
        h = torch.relu(x @ w1b)
        return h @ w2b

    h = torch.relu(x @ w1b)

    def dbwd():
        da = (dO @ w2b.t()) * (h > 0)
        return da @ w1b.t()

    fl = 2 * 2.0 * M * d * f
    for phase, fn in (("fwd", dfwd), ("bwd", dbwd)):
        ms = timer(fn, args.reps)
        rows.append(line("dense_mlp_cublas", phase, 0.0, ms, fl, peak, {"M": M, "d": d, "d_ff": f}))
    return rows


def sweep_attn(args, timer, peak):
    import torch

    from paper_2510_15964_b200 import block_sparse as BS, patterns as PT
    from oracle.sf_oracle import make_rng  # seeded PCG64 (sf/tensor_core.py:19-21) for the layouts only

    c = CFG2
    B, s, H, hd = c["B"], c["s"], c["H"], c["hd"]
    d = H * hd
    M = B * s
    g = torch.Generator(device="cuda").manual_seed(1)
    qkv = torch.randn(M, 3 * d, device="cuda", generator=g).to(torch.bfloat16)
    dO = (torch.randn(M, d, device="cuda", generator=g) * 0.1).to(torch.bfloat16)
    scale = 1.0 / np.sqrt(hd)
    rows = []
    for ab in args.attn_blk:
        n_b = s // ab
        dense_ms = {}
        for sp in [0.0] + args.sparsity:
            rng = make_rng(7)
            grids = np.zeros((H, n_b, n_b), bool)
            nnz = 0
            for h in range(H):
                cs = np.asarray(attn_layout(n_b, sp, rng))
                grids[h, cs[:, 0], cs[:, 1]] = True
                nnz += len(cs)
            dp = PT.DevicePool([f"h{h}" for h in range(H)], None, None, None, s, ab)
            tab = PT.tables128_from_grids(grids, s, ab)
            dp.tables = torch.from_numpy(tab).cuda()
            pidx = torch.arange(H, dtype=torch.int32, device="cuda")[None]
            Q, K, V = qkv[:, :d], qkv[:, d : 2 * d], qkv[:, 2 * d :]
            o = torch.empty(M, d, dtype=torch.bfloat16, device="cuda")
            st = {}

            def fwd():
                st["o"], st["lse"] = BS.attention_forward(Q, K, V, 3 * d, B, s, H, hd, pidx, 0, dp, scale, out=o)

            fwd()
            dqkv = torch.empty_like(qkv)

            def bwd():
                BS.attention_backward(Q, K, V, st["o"], dO, 3 * d, B, s, H, hd, pidx, 0, dp, scale, st["lse"],
                                      dqkv[:, :d], dqkv[:, d : 2 * d], dqkv[:, 2 * d :])

            # gathered 128x128 MMA tiles the kernels walk (forward / dQ and dK/dV), summed over heads
            work = [PT.tables128_work(tab, h) for h in range(H)]
            tiles_f, tiles_b = sum(w[0] for w in work), sum(w[1] for w in work)
            for phase, fn, mult in (("fwd", fwd, 4), ("bwd", bwd, 8)):
                ms = timer(fn, args.reps)
                if sp == 0.0:
                    dense_ms[phase] = ms
                fl = mult * B * nnz * ab * ab * hd  # nnz summed over heads
                rows.append(line("block_sparse_attn", phase, sp, ms, fl, peak, {
                    "attn_blk": ab, "n_b": n_b, "nnz_per_head": round(nnz / H, 1),
                    "density": round(nnz / (H * n_b * n_b), 4), "B": B, "s": s, "H": H, "hd": hd,
                    "mma_tiles_fwd_dq": tiles_f, "mma_tiles_dkdv": tiles_b, "dense_tiles": H * (-(-s // 128)) ** 2,
                    "speedup_vs_same_kernel_dense": round(dense_ms[phase] / ms, 3),
                    "kernels": "bsattn_fwd_tc" if phase == "fwd" else "bsattn_delta_tc + bsattn_dkdv_tc + bsattn_dq_tc"}))
    # dense SDPA (flash) of the same shape, non-causal
    import torch.nn.functional as F

    q = qkv[:, :d].reshape(B, s, H, hd).transpose(1, 2).contiguous().requires_grad_(True)
    k = qkv[:, d : 2 * d].reshape(B, s, H, hd).transpose(1, 2).contiguous().requires_grad_(True)
    v = qkv[:, 2 * d :].reshape(B, s, H, hd).transpose(1, 2).contiguous().requires_grad_(True)
    go = dO.reshape(B, s, H, hd).transpose(1, 2).contiguous()
    st = {}

    def sfwd():
        st["o"] = F.scaled_dot_product_attention(q, k, v)

    def sbwd():
        torch.autograd.grad(st["o"], (q, k, v), go, retain_graph=True)

    sfwd()
    for phase, fn, mult in (("fwd", sfwd, 4), ("bwd", sbwd, 8)):
        ms = timer(fn, args.reps)
        rows.append(line("dense_attn_sdpa", phase, 0.0, ms, mult * B * H * s * s * hd, peak,
                         {"B": B, "s": s, "H": H, "hd": hd}))
    return rows


def sweep_exposer(args, timer, peaks):
    """Exposer oracle mode (csrc/exposer.cu) at the cfg2 layer shape: exact block masses (fp32 dot
    products + float64 softmax: bound by the FP32/FP64 pipes, reported against the FP32 FFMA peak at
    the measured max clock), coverage selection, MLP block importance (HBM-bound: one read of z) and
    the whole OracleProvider per layer (cuBLAS projections included) next to PredictedProvider."""
    import torch

    from paper_2510_15964_b200 import exposer as EX, patterns as PT, predictor as P

    c = CFG2
    d, H, hd, f, s, B, blk = c["d"], c["H"], c["hd"], c["d_ff"], c["s"], c["B"], c["blk"]
    M = B * s
    fp32_peak = 148 * 128 * 2 * peaks.get("sm_max_mhz", 1965.0) * 1e6 / 1e12
    g = torch.Generator(device="cuda").manual_seed(0)
    qk = torch.randn(M, 2 * d, device="cuda", generator=g)
    z = torch.randn(M, f, device="cuda", generator=g)
    rows = []
    for ab in args.attn_blk:
        n_b = s // ab
        dp = P._pool_dev(PT.build_pool(n_b), torch.device("cuda"))
        ms = timer(lambda: EX.exact_block_mass(qk, B, s, H, n_b), args.reps)
        rows.append(line("exposer_exact_block_mass", "fwd", 0.0, ms, 2 * B * H * s * s * hd, fp32_peak,
                         {"n_b": n_b, "peak_kind": "fp32 FFMA", "exps_f64": 2 * B * H * s * s}))
        mass = EX.exact_block_mass(qk, B, s, H, n_b)
        for hs in (False, True):
            ms = timer(lambda: EX.select_by_coverage(mass, dp, 0.95, head_sum=hs), args.reps)
            print(json.dumps({"op": "exposer_select_by_coverage", "head_sum": hs, "n_b": n_b, "ms": round(ms, 4)}),
                  flush=True)
    ms = timer(lambda: EX.block_importance(z, B, s, blk), args.reps)
    gbs = M * f * 4 / (ms * 1e-3) / 1e9
    print(json.dumps({"op": "exposer_block_importance", "ms": round(ms, 4), "bytes": M * f * 4, "gbs": round(gbs, 1),
                      "frac_of_hbm": round(gbs / peaks["hbm"], 3)}), flush=True)
    imp = EX.block_importance(z, B, s, blk)
    ms = timer(lambda: EX.filter_neuron_blocks(imp, 0.1, blk), args.reps)
    print(json.dumps({"op": "exposer_filter_neuron_blocks", "ms": round(ms, 4)}), flush=True)
    return rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--ops", default="mlp,attn")
    ap.add_argument("--sparsity", default="0.5,0.75,0.9")
    ap.add_argument("--attn-blk", default="16,64,128")
    args = ap.parse_args()
    args.sparsity = [float(x) for x in args.sparsity.split(",")]
    args.attn_blk = [int(x) for x in args.attn_blk.split(",")]
    import torch

    from bench import load_peaks
    from paper_2510_15964_b200 import _abi

    _abi.lib()
    torch.cuda.set_device(0)
    peaks = load_peaks()
    peak = peaks["bf16"]  # kernels timed alone: burst peak
    print(json.dumps({"sweep": "cfg2 isolated operators, OPT-1.3B layer shapes", **CFG2, "peak_tflops": peak,
                      "peak_src": f"{peaks['src']} burst bf16", "gpu": torch.cuda.get_device_name(0)}), flush=True)
    timer = Timer()
    ops = args.ops.split(",")
    if "mlp" in ops:
        sweep_mlp(args, timer, peak)
    if "attn" in ops:
        sweep_attn(args, timer, peak)
    if "exposer" in ops:
        sweep_exposer(args, timer, peaks)


if __name__ == "__main__":
    main()
