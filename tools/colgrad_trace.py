"""Phase timeline (clock64) of colgrad_partial at the cfg3 dense shape (M=4096, 2048 columns, r=8)."""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2510_15964_b200 import _abi, neuron_ops as N  # noqa: E402

B, s, d, r = 8, 512, 2048, 8
dev = torch.device("cuda")
x = torch.randn(B * s, d, device=dev).to(torch.bfloat16)
p = torch.randn(B * s, r, device=dev)
G = torch.empty(r, d, device=dev)
lib = _abi.lib()
lib.lx_debug_set_colgrad_trace.argtypes = [ctypes.c_void_p]
for _ in range(3):
    N.colgrad(p, x, B, s, d, r, 1.0, G, d, 1)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(20):
    N.colgrad(p, x, B, s, d, r, 1.0, G, d, 1)
b.record()
torch.cuda.synchronize()
print(f"colgrad (partial + final) {a.elapsed_time(b) / 20 * 1e3:.1f} us/call, {x.numel() * 2 / 1e6:.1f} MB of X")
buf = torch.zeros(2048, 8, dtype=torch.int64, device=dev)
lib.lx_debug_set_colgrad_trace(buf.data_ptr())
N.colgrad(p, x, B, s, d, r, 1.0, G, d, 1)
torch.cuda.synchronize()
lib.lx_debug_set_colgrad_trace(None)
t = buf.cpu().numpy().astype(np.int64)
t = t[t[:, 0] > 0]
rel = t - t[:, :1]
print(f"{len(t)} CTAs; mean cycles from start: P staged {rel[:, 1].mean():.0f}, first tile {rel[:, 2].mean():.0f}, "
      f"last tile done {rel[:, 3].mean():.0f}, end {rel[:, 4].mean():.0f}; start spread {t[:, 0].max() - t[:, 0].min()}")
