"""fc1/fc2 gather GEMM time vs neuron block size at fixed density (TMA box count experiment)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2510_15964_b200 import _abi  # noqa: E402

B, s, d, f = 8, 512, 2048, 8192
st = _abi.stream_handle()
x = torch.randn(B * s, d, device="cuda").bfloat16()
w1t = torch.randn(f, d, device="cuda").bfloat16()
w2 = torch.randn(f, d, device="cuda").bfloat16()
a = torch.randn(B * s, f, device="cuda").bfloat16()
out = torch.empty(B * s, f, device="cuda").bfloat16()
o2 = torch.empty(B * s, d, device="cuda").bfloat16()


def timeit(fn, n=10):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


for dens in (0.15, 1.0):
    for blk in (16, 32, 64):
        n_blk = f // blk
        act = np.sort(np.random.default_rng(0).permutation(n_blk)[: max(1, int(dens * n_blk))])
        counts = torch.full((B,), len(act), dtype=torch.int32, device="cuda")
        ids = torch.zeros(B, n_blk, dtype=torch.int32, device="cuda")
        ids[:, : len(act)] = torch.from_numpy(act).cuda().int()
        fl = 2 * B * s * d * len(act) * blk
        t1 = timeit(lambda: _abi.call("lx_neuron_fc1", x.data_ptr(), B, s, d, f, blk, w1t.data_ptr(), counts.data_ptr(), ids.data_ptr(), None, None, None, 0, 1.0, 1, out.data_ptr(), f, None, st))
        t2 = timeit(lambda: _abi.call("lx_neuron_fc2", a.data_ptr(), f, B, s, d, f, blk, w2.data_ptr(), counts.data_ptr(), ids.data_ptr(), None, None, None, 0, 1.0, o2.data_ptr(), 0, None, None, st))
        print(f"density {dens} blk {blk}: fc1 {t1:.4f} ms {fl / t1 / 1e9:.0f} TF/s | fc2 {t2:.4f} ms {fl / t2 / 1e9:.0f} TF/s")
