"""One launch each of cuBLAS and lx_linear (modes from argv) at the cfg3 QKV projection shape, for ncu."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2510_15964_b200 import _abi, model as M  # noqa: E402

Mr, K, N = 4096, 2048, 6144
a = torch.randn(Mr, K, device="cuda").bfloat16()
bt = torch.randn(N, K, device="cuda").bfloat16()
torch.mm(a, bt.t())
for mode in [int(x) for x in sys.argv[1:]] or [0, 1]:
    _abi.lib().lx_gemm_set_cta_pair(mode)
    M.linear(a, bt)
torch.cuda.synchronize()
