"""The four cfg3 projection GEMMs on lx_linear (fused epilogue) vs cuBLAS bf16 (torch.mm), CUDA-event timed."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2510_15964_b200 import _abi, model as M  # noqa: E402

M_, d = 4096, 2048


def t(fn, n=20):
    for _ in range(3):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


cases = {"qkv": (d, 3 * d, 16, False), "o_proj": (d, d, 0, True), "d_heads": (d, d, 0, False), "dx": (3 * d, d, 16, False),
         "lm_head": (d, 50272, 0, False)}
modes = [int(x) for x in sys.argv[1:]] or [0, 5]
for name, (K, N, r, resid) in cases.items():
    a = torch.randn(M_, K, device="cuda").bfloat16()
    bt = torch.randn(N, K, device="cuda").bfloat16()
    bias = torch.randn(N, device="cuda")
    lx = torch.randn(M_, max(r, 1), device="cuda") if r else None
    lw = torch.randn(max(r, 1), N, device="cuda") if r else None
    res = torch.randn(M_, N, device="cuda") if resid else None
    fl = 2 * M_ * N * K
    w = bt.t()
    msc = t(lambda: torch.mm(a, w))
    ref = torch.mm(a, w).float()
    line = f"{name:8s} M={M_} N={N} K={K}: cuBLAS {msc * 1e3:7.1f} us {fl / msc / 1e9:6.0f} TF/s"
    for mode in modes:
        _abi.lib().lx_gemm_set_cta_pair(mode)
        ms = t(lambda: M.linear(a, bt, out_f32=resid, resid=res, bias=bias, lora_x=lx, lora_w=lw, w_sr=N, w_sc=1, r=r))
        ms0 = t(lambda: M.linear(a, bt))
        wkn = bt.t().contiguous()
        mskn = t(lambda: M.linear(a, wkn, kn=True))
        err = ((M.linear(a, bt).float() - ref).abs().max() / ref.abs().max()).item()
        errkn = ((M.linear(a, wkn, kn=True).float() - ref).abs().max() / ref.abs().max()).item()
        line += (f" | m{mode}: fused {ms * 1e3:6.1f} plain {ms0 * 1e3:6.1f} us {fl / ms0 / 1e9:5.0f} TF/s err {err:.1e}"
                 f" kn {mskn * 1e3:6.1f} us err {errkn:.1e}")
    _abi.lib().lx_gemm_set_cta_pair(0)
    print(line, flush=True)
