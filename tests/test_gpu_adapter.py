"""The fp32 adapter kernels (csrc/adapter.cu) against the reference algebra (sf/model.py:315-319,
sf/autograd.py:69-75) evaluated in float64 on the same inputs: forward output, pre-activation, input gradient
and all four parameter gradients within 1e-5 (fp32 accumulation), deterministic across runs."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    return torch.device("cuda")


def rel(a, b):
    a, b = a.detach().double().cpu(), b.detach().double().cpu()
    return float((a - b).abs().max() / b.abs().max().clamp_min(1e-30))


@pytest.mark.parametrize("M,d,r", [(1, 64, 8), (300, 768, 8), (4096, 2048, 8), (257, 4096, 16), (96, 5120, 8)])
def test_adapter_kernels_match_float64(dev, M, d, r):
    from paper_2510_15964_b200 import autograd as AG, model as M_

    g = torch.Generator(device="cpu").manual_seed(M + d)
    x = torch.randn(M, d, generator=g).to(dev)
    ad = M_.AdapterLayer(*(t.to(dev) for t in (torch.randn(d, r, generator=g) * 0.05, torch.randn(r, generator=g) * 0.1,
                                               torch.randn(r, d, generator=g) * 0.05, torch.randn(d, generator=g) * 0.1)))
    dy = torch.randn(M, d, generator=g).to(dev)
    out, cache = M_.adapter_forward(x, ad)
    grads = {}
    dx = AG.adapter_backward(dy, ad, cache, grads, "a")
    torch.cuda.synchronize()
    X, Wd, bd, Wu, bu, DY = (t.double() for t in (x, ad.w_down, ad.b_down, ad.w_up, ad.b_up, dy))
    z = X @ Wd + bd
    h = z.clamp_min(0)
    assert rel(cache["z"], z) < 1e-5
    assert rel(out, X + h @ Wu + bu) < 1e-5
    dh = (DY @ Wu.t()) * (z > 0)
    assert rel(dx, DY + dh @ Wd.t()) < 1e-5
    assert rel(grads["a.w_up"], h.t() @ DY) < 1e-5
    assert rel(grads["a.b_up"], DY.sum(0)) < 1e-5
    assert rel(grads["a.w_down"], X.t() @ dh) < 1e-5
    assert rel(grads["a.b_down"], dh.sum(0)) < 1e-5
    res = torch.randn(M, d, generator=g).to(dev)
    out_r, _ = M_.adapter_forward(x, ad, resid=res)  # fused residual add: bitwise resid + out
    torch.cuda.synchronize()
    assert torch.equal(out_r, res + out)
    grads2 = {}
    AG.adapter_backward(dy, ad, cache, grads2, "a")
    for k in grads:
        assert torch.equal(grads[k], grads2[k]), k
