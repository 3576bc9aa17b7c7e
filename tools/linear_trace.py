"""Phase timeline of the dense lx_linear engine (clock64 stamps, lx_debug_set_gemm_trace) vs cuBLAS, for the cfg3
projection shapes: per-CTA start -> first stage landed, mainloop per tile, epilogue, and the event-timed launch."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2510_15964_b200 import _abi, model as M  # noqa: E402

dev = torch.device("cuda")
buf = torch.zeros(160, 32, dtype=torch.int64, device=dev)


def timed(fn, n=20):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


for (Mr, N, K) in ((4096, 2048, 2048), (4096, 6144, 2048), (4096, 2048, 6144)):
    a = torch.randn(Mr, K, device=dev).bfloat16()
    bt = torch.randn(N, K, device=dev).bfloat16()
    bias = torch.randn(N, device=dev)
    w = bt.t()
    cu = timed(lambda: torch.mm(a, w))
    us = timed(lambda: M.linear(a, bt))
    usb = timed(lambda: M.linear(a, bt, bias=bias))
    buf.zero_()
    _abi.call("lx_debug_set_gemm_trace", buf.data_ptr())
    M.linear(a, bt)
    torch.cuda.synchronize()
    _abi.call("lx_debug_set_gemm_trace", None)
    t = buf.cpu().numpy().astype(np.int64)[:148]
    lead = t[:, 2] > 0
    r = t[lead] - t[lead, 0:1]
    print(f"M={Mr} N={N} K={K}: cuBLAS {cu:.1f} us, lx_linear {us:.1f} us (+bias {usb:.1f}); leaders {lead.sum()}")
    for i in range(3):
        sel = r[:, 2 + 4 * i] > 0
        if not sel.any():
            continue
        q = r[sel]
        print(f"   tile{i}: first stage {q[:, 2 + 4 * i].mean():7.0f}  last MMA {q[:, 3 + 4 * i].mean():7.0f}  "
              f"epi start {q[:, 4 + 4 * i].mean():7.0f}  epi end {q[:, 5 + 4 * i].mean():7.0f}  (n={sel.sum()})")
    print(f"   end {r[:, 1].mean():7.0f} (max {r[:, 1].max()}) cycles")
