"""Which pool patterns does the device predictor choose in bench.py's cfg3 workload? Per layer, the
pattern histogram of the calibrated local heads and of the remaining heads, plus score-map statistics
of one local head (diagonal vs off-diagonal of the binarised m x m map). Diagnostics only."""
import sys
from collections import Counter
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2510_15964_b200 import exposer as EX, model as M, predictor as P  # noqa: E402
from paper_2510_15964_b200.engine import FinetuneEngine  # noqa: E402

cfg = dict(bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg3"])
lf = float(sys.argv[2]) if len(sys.argv) > 2 else 0.75
dev = torch.device("cuda")
model, state, prov = bench.build_workload(cfg, dev, 0, 0.85, lf)
eng = FinetuneEngine(model, state, prov, lr=1e-4)
tok = torch.randint(0, cfg["V"], (cfg["B"], cfg["s"] + 1), generator=torch.Generator().manual_seed(2)).to(dev)
eng.step(tok)
torch.cuda.synchronize()
ids = list(model.pool)
H = cfg["H"]
nl = int(round(H * lf))
print("achieved", bench.achieved_sparsity(eng.last_masks, model))
if "-v" in sys.argv:
    for layer, lm in enumerate(eng.last_masks):
        hp = lm.head_patterns.cpu().numpy()
        loc = Counter(ids[i] for i in hp[:, :nl].ravel())
        oth = Counter(ids[i] for i in hp[:, nl:].ravel())
        print(f"layer {layer:2d} local {dict(loc)} other {dict(oth)}")
sys.exit(0)
# score maps of layer L/2 local head 0 on the recorded LN1 rows
rec = EX._Recorder(model)
with torch.no_grad():
    M.model_forward(model, tok[:, :-1], rec)
for layer in (0, cfg["L"] // 2, cfg["L"] - 1):
    xs, m = P.x_small_of(rec.h_attn[layer])
    idx, sc = P.attn_pattern_idx(xs, cfg["B"], m, prov.predictors["attn"][layer], model.dpool, model.dims.n_b,
                                 prov.pcfg, dump=True)
    s0 = sc[0, 0].cpu().numpy()
    act = s0 > 0.5 * s0.max()
    print(f"layer {layer}: head0 map max {s0.max():.3g} diag mean {np.diag(s0).mean():.3g} offdiag max "
          f"{(s0 - np.diag(np.diag(s0))).max():.3g} min diag {np.diag(s0).min():.3g}; active cells {int(act.sum())} "
          f"(diag {int(np.diag(act).sum())}); pattern {ids[int(idx[0, 0])]}")
