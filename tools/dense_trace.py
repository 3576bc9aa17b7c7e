"""Dense lx_linear timeline (clock64 stamps, see gemm_trace.py) per GEMM engine: effective SM clock under
load (CTA lifetime cycles / event-timed duration) and mainloop cycles per K stage, vs cuBLAS time."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2510_15964_b200 import _abi, model as M  # noqa: E402

Mr, K, N = 4096, 2048, int(sys.argv[1]) if len(sys.argv) > 1 else 6144
dev = torch.device("cuda")
a = torch.randn(Mr, K, device=dev).bfloat16()
bt = torch.randn(N, K, device=dev).bfloat16()
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


w = bt.t()
print(f"M={Mr} N={N} K={K}: cuBLAS {timed(lambda: torch.mm(a, w)):.1f} us")
for mode in [int(x) for x in sys.argv[2:]] or [0, 1, 4]:
    _abi.lib().lx_gemm_set_cta_pair(mode)
    us = timed(lambda: M.linear(a, bt))
    buf.zero_()
    _abi.call("lx_debug_set_gemm_trace", buf.data_ptr())
    M.linear(a, bt)
    torch.cuda.synchronize()
    _abi.call("lx_debug_set_gemm_trace", None)
    t = buf.cpu().numpy().astype(np.int64)[:148]
    ok = t[:, 1] > 0
    life = (t[ok, 1] - t[ok, 0])
    lead = t[:, 2] > 0
    st = (t[lead, 7] - t[lead, 6]) / (K / 64)  # tile 1: first stage -> last MMA issued
    epi = (t[lead, 8 + 1] - t[lead, 8]) if lead.any() else np.zeros(1)
    print(f"  mode {mode}: {us:.1f} us; lifetime {life.mean():.0f} cyc (max {life.max()}) -> {life.max() / us:.0f} MHz; "
          f"tile1 mainloop {st.mean():.0f} cyc/stage; tile1 epi {epi.mean():.0f} cyc; CTAs {ok.sum()} leaders {lead.sum()}",
          flush=True)
_abi.lib().lx_gemm_set_cta_pair(0)
