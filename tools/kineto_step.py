"""Warm, non-serialised per-kernel device times of one cfg3 step (torch.profiler / CUPTI).

    python tools/kineto_step.py [cfg3] [--graph] > gpurun_out/kineto.txt

Eager by default (kernel durations as in the graph, host gaps excluded from the sums); with --graph
the captured step is replayed under the profiler. Prints the per-kernel totals and the per-launch
sequence of one layer so kernel shares can be compared against the ncu (cold, serialised) list.
"""
import collections
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402
from paper_2510_15964_b200.engine import FinetuneEngine  # noqa: E402

args = [a for i, a in enumerate(sys.argv[1:]) if not a.startswith("--") and not a.isdigit() and sys.argv[i] != "--peft"]
cfg = bench.CONFIGS[args[0] if args else "cfg3"]
graph = "--graph" in sys.argv
dev = torch.device("cuda", 0)
if "--pair" in sys.argv:  # GEMM engine variant (lx_gemm_set_cta_pair): 0 single CTA, 1 pairs 256x256, 2 pairs 256x128
    from paper_2510_15964_b200 import _abi

    _abi.lib().lx_gemm_set_cta_pair(int(sys.argv[sys.argv.index("--pair") + 1]))
peft = sys.argv[sys.argv.index("--peft") + 1] if "--peft" in sys.argv else "lora"
model, state, prov = bench.build_workload(cfg, dev, 0, 0.85, 0.75, peft=peft)
eng = FinetuneEngine(model, state, prov, lr=1e-4)
tok = torch.randint(0, cfg["V"], (cfg["B"], cfg["s"] + 1), device=dev)
if graph:
    eng.capture(tok)
    for _ in range(3):
        eng.replay()
else:
    for _ in range(3):
        eng.step(tok)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    if graph:
        eng.replay()
    else:
        eng.step(tok)
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)
agg = collections.defaultdict(lambda: [0, 0.0])
busy = 0.0
for e in evs:
    d = e.time_range.end - e.time_range.start
    k = e.name.split("(")[0][:90]
    agg[k][0] += 1
    agg[k][1] += d
    busy += d
span = evs[-1].time_range.end - evs[0].time_range.start if evs else 0
print(f"{'graph' if graph else 'eager'} step: {len(evs)} kernels, device busy {busy / 1e3:.3f} ms, span {span / 1e3:.3f} ms")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:45]:
    print(f"{t / 1e3:8.3f} ms {100 * t / busy:5.1f}%  n={n:4d}  {t / n:8.1f} us/launch  {k}")
# one middle layer's forward and backward launch sequence (with gaps)
print("\nlaunch sequence (us: start offset, duration, gap before):")
prev_end = None
t0 = evs[0].time_range.start if evs else 0
for e in evs:
    gap = (e.time_range.start - prev_end) if prev_end is not None else 0
    prev_end = e.time_range.end
    print(f"{(e.time_range.start - t0):10.1f} {e.time_range.end - e.time_range.start:8.1f} {gap:7.1f}  {e.name[:80]}")
