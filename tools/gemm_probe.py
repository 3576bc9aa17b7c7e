"""cfg3-shaped MLP GEMMs in isolation (for ncu --set full): fc1 N-gather, fc2 K-gather, dense."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2510_15964_b200 import _abi  # noqa: E402

B, s, d, f, blk = 8, 512, 2048, 8192, 16
dens = float(sys.argv[1]) if len(sys.argv) > 1 else 0.15
n_blk = f // blk
rng = np.random.default_rng(0)
act = np.sort(rng.permutation(n_blk)[: int(dens * n_blk)])
counts = torch.full((B,), len(act), dtype=torch.int32, device="cuda")
ids = torch.zeros(B, n_blk, dtype=torch.int32, device="cuda")
ids[:, : len(act)] = torch.from_numpy(act).cuda().int()
x = torch.randn(B * s, d, device="cuda").bfloat16()
w1t = torch.randn(f, d, device="cuda").bfloat16()
w2 = torch.randn(f, d, device="cuda").bfloat16()
a = torch.randn(B * s, f, device="cuda").bfloat16()
out = torch.empty(B * s, f, device="cuda").bfloat16()
o2 = torch.empty(B * s, d, device="cuda").bfloat16()
c = torch.empty(B * s, f, device="cuda", dtype=torch.float32)
st = _abi.stream_handle()
for _ in range(3):
    _abi.call("lx_neuron_fc1", x.data_ptr(), B, s, d, f, blk, w1t.data_ptr(), counts.data_ptr(), ids.data_ptr(), None, None,
              None, 0, 1.0, 1, out.data_ptr(), f, None, st)
    _abi.call("lx_neuron_fc2", a.data_ptr(), f, B, s, d, f, blk, w2.data_ptr(), counts.data_ptr(), ids.data_ptr(), None, None,
              None, 0, 1.0, o2.data_ptr(), 0, None, None, st)
    _abi.call("lx_gemm_bf16_tn", x.data_ptr(), d, w1t.data_ptr(), d, out.data_ptr(), f, 0, B * s, f, d, 0, st)
torch.cuda.synchronize()
for name, fn, flops in (("fc1", lambda: _abi.call("lx_neuron_fc1", x.data_ptr(), B, s, d, f, blk, w1t.data_ptr(), counts.data_ptr(), ids.data_ptr(), None, None, None, 0, 1.0, 1, out.data_ptr(), f, None, st), 2 * B * s * d * len(act) * blk),
                        ("fc2", lambda: _abi.call("lx_neuron_fc2", a.data_ptr(), f, B, s, d, f, blk, w2.data_ptr(), counts.data_ptr(), ids.data_ptr(), None, None, None, 0, 1.0, o2.data_ptr(), 0, None, None, st), 2 * B * s * d * len(act) * blk),
                        ("dense", lambda: _abi.call("lx_gemm_bf16_tn", x.data_ptr(), d, w1t.data_ptr(), d, out.data_ptr(), f, 0, B * s, f, d, 0, st), 2 * B * s * d * f)):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"{name}: {ms:.4f} ms  {flops / ms / 1e9:.1f} TFLOP/s")
ref = torch.empty(B * s, f, device="cuda").bfloat16()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    torch.mm(x, w1t.t(), out=ref)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"cublas dense: {ms:.4f} ms  {2 * B * s * d * f / ms / 1e9:.1f} TFLOP/s")
