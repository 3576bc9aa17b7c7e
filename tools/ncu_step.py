"""One cfg3 training step (eager) bracketed by cudaProfilerStart/Stop for ncu --profile-from-start off:
    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
        --profile-from-start off --csv python tools/ncu_step.py [cfg3]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2510_15964_b200.engine import FinetuneEngine  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg3"]
dev = torch.device("cuda", 0)
model, state, prov = bench.build_workload(cfg, dev, 0, 0.85, 0.75)
eng = FinetuneEngine(model, state, prov, lr=1e-4)
tok = torch.randint(0, cfg["V"], (cfg["B"], cfg["s"] + 1), generator=torch.Generator().manual_seed(2)).to(dev)
for _ in range(2):
    eng.step(tok)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
eng.step(tok)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
