"""Phase timeline (clock64) of the MLP GEMMs at cfg3 layer shapes, both engine variants.
Stamps per CTA: 0 start, 1 end, then per tile i<3: 2+4i first stage landed (MMA), 3+4i last MMA
issued, 4+4i epilogue got the accumulator, 5+4i epilogue done."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2510_15964_b200 import _abi, neuron_ops as N  # noqa: E402

B, s, d, f, blk, dens = 8, 512, 2048, 8192, 16, float(sys.argv[1]) if len(sys.argv) > 1 else 0.15
dev = torch.device("cuda")
g = torch.Generator().manual_seed(0)
masks = torch.rand(B, f // blk, generator=g) < dens
nm = N.lower_mask(masks.to(dev), f // blk, blk, B, dev)
x = (torch.randn(B * s, d, device=dev) * 0.5).to(torch.bfloat16)
w1t = (torch.randn(f, d, device=dev) * 0.02).to(torch.bfloat16)
w2 = (torch.randn(f, d, device=dev) * 0.02).to(torch.bfloat16)
w1p, w2p = N.pack_active_rows(w1t, nm), N.pack_active_rows(w2, nm)
h = torch.empty(B * s, f, device=dev, dtype=torch.bfloat16)
out = torch.empty(B * s, d, device=dev, dtype=torch.bfloat16)
resid = torch.randn(B * s, d, device=dev)
st = _abi.stream_handle()
buf = torch.zeros(160, 32, dtype=torch.int64, device=dev)
bits = torch.zeros(B * s, f // 16, dtype=torch.int16, device=dev)


def fc1():
    _abi.call("lx_neuron_fc1", x.data_ptr(), B, s, d, f, blk, w1t.data_ptr(), nm.counts.data_ptr(), nm.ids.data_ptr(),
              None, None, None, 0, 1.0, 1, h.data_ptr(), f, w1p.data_ptr(), bits.data_ptr() if "--bits" in sys.argv else None,
              st)


def fc2():
    _abi.call("lx_neuron_fc2", h.data_ptr(), f, B, s, d, f, blk, w2.data_ptr(), nm.counts.data_ptr(), nm.ids.data_ptr(),
              None, None, None, 0, 1.0, out.data_ptr(), 0, None, w2p.data_ptr(), st)


dz = torch.empty(B * s, f, device=dev, dtype=torch.bfloat16)
dxo = torch.empty(B * s, d, device=dev, dtype=torch.bfloat16)


def fc2_dgrad():  # dz = (dO W2[cols]^T) * relu'(a), a = fc1's output h
    _abi.call("lx_neuron_fc2_dgrad", out.data_ptr(), B, s, d, f, blk, w2.data_ptr(), nm.counts.data_ptr(),
              nm.ids.data_ptr(), None, None, 0, h.data_ptr(), dz.data_ptr(), f, w2p.data_ptr(),
              bits.data_ptr() if "--bits" in sys.argv else None, st)


def fc1_dgrad():  # dx = dz W1[:, cols]^T
    _abi.call("lx_neuron_fc1_dgrad", dz.data_ptr(), f, B, s, d, f, blk, w1t.data_ptr(), nm.counts.data_ptr(),
              nm.ids.data_ptr(), None, None, 0, dxo.data_ptr(), 0, w1p.data_ptr(), st)


for pair in ((0,) if "--default" in sys.argv else (2, 1, 0)):
    _abi.lib().lx_gemm_set_cta_pair(pair)
    for name, fn in (("fc1", fc1), ("fc2", fc2), ("fc2_dgrad", fc2_dgrad), ("fc1_dgrad", fc1_dgrad)):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20):
            fn()
        b.record()
        torch.cuda.synchronize()
        us = a.elapsed_time(b) / 20 * 1e3
        gr = torch.cuda.CUDAGraph()  # device-side per-launch time (no host launch overhead)
        s2 = torch.cuda.Stream()
        s2.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s2):
            st_prev = st
            globals()["st"] = _abi.stream_handle()
            with torch.cuda.graph(gr, stream=s2):
                for _ in range(20):
                    fn()
            globals()["st"] = st_prev
        torch.cuda.current_stream().wait_stream(s2)
        gr.replay()
        torch.cuda.synchronize()
        a.record()
        gr.replay()
        b.record()
        torch.cuda.synchronize()
        us_graph = a.elapsed_time(b) / 20 * 1e3
        buf.zero_()
        _abi.call("lx_debug_set_gemm_trace", buf.data_ptr())
        fn()
        torch.cuda.synchronize()
        _abi.call("lx_debug_set_gemm_trace", None)
        t = buf.cpu().numpy().astype(np.int64)[:148]
        act = t[:, 2] > 0
        base = t[:, 0:1]
        rel = np.where(t > 0, t - base, 0)
        print(f"{name} pair={pair}: {us:.1f} us/launch (graph {us_graph:.1f}), CTAs with a tile {act.sum()}; lifetime mean "
              f"{(t[:, 1] - t[:, 0]).mean():.0f} cyc")
        pro = [np.median(rel[act, k]) for k in (14, 15, 16, 17)]
        print(f"   prologue: pdl wait {pro[0]:.0f}  counts {pro[1]:.0f}  width/prefix {pro[2]:.0f}  cluster sync {pro[3]:.0f}")
        for i in range(2):
            sel = t[:, 2 + 4 * i] > 0
            if not sel.any():
                continue
            r = rel[sel]
            print(f"   tile{i}: first stage {r[:, 2 + 4 * i].mean():7.0f}  last MMA {r[:, 3 + 4 * i].mean():7.0f}  "
                  f"epi start {r[:, 4 + 4 * i].mean():7.0f}  epi end {r[:, 5 + 4 * i].mean():7.0f}  (n={sel.sum()})")
_abi.lib().lx_gemm_set_cta_pair(0)
