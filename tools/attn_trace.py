"""Phase timeline of the tcgen05 attention forward at cfg3 layer shapes (debug stamps, clock64).
Prints the mean cycles between phases per CTA and the SM-level CTA overlap."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2510_15964_b200 import _abi, patterns as PT  # noqa: E402

B, s, H, hd, ab = 8, 512, 32, 64, 64
d = H * hd
dev = torch.device("cuda")
qkv = (torch.randn(B * s, 3 * d, device=dev) * 0.5).to(torch.bfloat16)
pool = PT.build_pool(s // ab)
dp = PT.device_pool(pool, dev, s, ab)
dense = list(pool).index("dense")
pidx = torch.full((B, H), dense, dtype=torch.int32, device=dev)
o = torch.empty(B * s, d, dtype=torch.bfloat16, device=dev)
lse = torch.empty(B, H, s, device=dev)
n_cta = (s // 128) * H * B
buf = torch.zeros(n_cta, 32, dtype=torch.int64, device=dev)


def run():
    _abi.call("lx_bsattn_fwd_tc", qkv.data_ptr(), 3 * d, B, s, H, hd, pidx.data_ptr(), H, dp.tables.data_ptr(),
              dp.gather_rows, 1.0 / 8, o.data_ptr(), d, lse.data_ptr(), _abi.stream_handle())


for _ in range(3):
    run()
torch.cuda.synchronize()
st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
st.record()
for _ in range(10):
    run()
en.record()
torch.cuda.synchronize()
print(f"fwd {st.elapsed_time(en) / 10 * 1e3:.1f} us per launch ({n_cta} CTAs, dense pattern)")
_abi.call("lx_debug_set_attn_trace", buf.data_ptr())
run()
torch.cuda.synchronize()
_abi.call("lx_debug_set_attn_trace", None)
t = buf.cpu().numpy().astype(np.int64)
names = {0: "start", 1: "setup", 2: "q_full", 4: "kv0", 5: "kv1", 6: "kv2", 7: "kv3", 8: "s0", 9: "s1", 10: "s2", 11: "s3",
         12: "p0", 13: "p1", 14: "p2", 15: "p3", 16: "o_done", 17: "epi_end", 18: "dealloc"}
order = [0, 1, 2, 4, 8, 12, 5, 9, 13, 6, 10, 14, 7, 11, 15, 16, 17, 18]
prev = 0
for k in order[1:]:
    dlt = t[:, k] - t[:, prev]
    print(f"{names[prev]:>8s} -> {names[k]:<8s} mean {dlt.mean():8.0f}  p50 {np.median(dlt):8.0f}  cycles")
    prev = k
tot = t[:, 18] - t[:, 0]
print(f"CTA lifetime mean {tot.mean():.0f} cycles")
sm = t[:, 31]
span = []
for i in np.unique(sm):
    sel = sm == i
    span.append(t[sel, 18].max() - t[sel, 0].min())
print(f"per-SM busy span mean {np.mean(span):.0f} cycles, CTAs/SM {n_cta / len(np.unique(sm)):.1f}; "
      f"sum of CTA lifetimes / span = {np.mean([tot[sm == i].sum() / sp for i, sp in zip(np.unique(sm), span)]):.2f}")
