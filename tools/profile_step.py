"""One eager cfg3 fine-tune step bracketed by cudaProfilerStart/Stop (for `ncu --profile-from-start off`)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2510_15964_b200.engine import FinetuneEngine  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg3"]
dev = torch.device("cuda", 0)
model, state, prov = bench.build_workload(cfg, dev, 0, 0.85, 0.5)
eng = FinetuneEngine(model, state, prov, lr=1e-4)
tok = torch.randint(0, cfg["V"], (cfg["B"], cfg["s"] + 1), device=dev)
for _ in range(2):
    eng.step(tok)
torch.cuda.synchronize()
torch.cuda.profiler.start()
eng.step(tok)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("done")
