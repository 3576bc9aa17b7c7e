"""CPU checks of the drop-in boundary: the C-ABI library loads without a GPU and
exports every symbol include/sparseft_b200.h declares; the ctypes table covers
them all; error codes map to the reference exception types."""

import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def header_symbols():
    text = (ROOT / "include" / "sparseft_b200.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int|long long|size_t|const char\*)\s+(lx_\w+)\s*\(", text, re.M)))


def test_header_declares_entry_points():
    syms = header_symbols()
    assert "lx_neuron_fc1" in syms and "lx_bsattn_bwd_tc" in syms and "lx_predict_mlp_mask" in syms
    assert len(syms) >= 20


def test_library_exports_every_header_symbol():
    from paper_2510_15964_b200 import _abi

    if not _abi.LIB_PATH.exists():
        pytest.skip("extension not built (run __graft_entry__.build())")
    lib = _abi.lib()
    missing = [s for s in header_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert set(header_symbols()) == set(_abi.SIGNATURES), "ctypes table out of sync with the header"
    assert lib.lx_abi_version() == 1


def test_error_mapping_without_gpu():
    """A shape error is raised before any CUDA call, as the reference's ValueError subclasses."""
    from paper_2510_15964_b200 import _abi, errors as E

    if not _abi.LIB_PATH.exists():
        pytest.skip("extension not built")
    with pytest.raises(E.UnsupportedError):
        _abi.call("lx_neuron_fc1", None, 1, 16, 64, 64, 24, None, None, None, None, None, None, 0, 1.0, 1, None, 64, None,
                  None, None)
    with pytest.raises(E.LayoutError):  # gather_rows must be a power of two in [16, 128]
        _abi.call("lx_bsattn_fwd_tc", None, 192, 1, 128, 1, 64, None, 0, None, 48, 0.125, None, 64, None, None)
    assert issubclass(E.LayoutError, ValueError) and issubclass(E.MaskError, ValueError)


def test_integration_bindings_match_the_abi_table():
    """Every ctypes binding shown in INTEGRATION.md has the argument types of the package's own table."""
    from paper_2510_15964_b200 import _abi

    text = (ROOT / "INTEGRATION.md").read_text()
    alias = {"P": _abi._P, "I": _abi._I, "F": _abi._F, "D": _abi._D, "C.c_longlong": _abi._LL}
    found = re.findall(r"_lib\.(lx_\w+)\.argtypes = \[([^\]]*)\]", text)
    assert len(found) >= 10
    for name, args in found:
        types = [alias[a.strip()] for a in args.split(",")]
        assert types == list(_abi.SIGNATURES[name]), name


def test_bench_counts_every_kernel_call_of_the_step():
    """bench.py's gpu_launches counts kernels per C-ABI call: every entry point the fine-tune step calls
    (engine, model, autograd, neuron_ops, predictor, block_sparse, dp) has a kernel count."""
    import bench

    names = set()
    for mod in ("engine", "model", "autograd", "neuron_ops", "predictor", "block_sparse", "dp"):
        names |= set(re.findall(r'_abi\.call\(\s*"(lx_\w+)"', (ROOT / "paper_2510_15964_b200" / f"{mod}.py").read_text()))
    debug = {"lx_debug_set_gemm_trace", "lx_debug_set_attn_trace"}
    missing = sorted(n for n in names - debug if n not in bench.KERNELS_PER_CALL)
    assert not missing, missing
