"""ctypes binding of the C-ABI (include/sparseft_b200.h).

Loads the in-tree `libsparseft_b200.so`. There is no fallback: if the library
is missing or no sm_100 GPU is present, calls raise immediately.
"""

from __future__ import annotations

import ctypes as C
from pathlib import Path

from . import errors as E

import os

# LX_LIB: an alternative build of the same library (experiments only; tests record which .so loaded)
LIB_PATH = Path(os.environ.get("LX_LIB") or Path(__file__).resolve().parent / "libsparseft_b200.so")

_P = C.c_void_p
_I = C.c_int
_F = C.c_float
_D = C.c_double
_LL = C.c_longlong

# symbol -> argtypes (order as declared in include/sparseft_b200.h)
SIGNATURES: dict[str, list] = {
    "lx_last_error": [],
    "lx_abi_version": [],
    "lx_device_sm_count": [],
    "lx_gemm_set_cta_pair": [_I],
    "lx_debug_set_gemm_trace": [_P],
    "lx_gemm_bf16_tn": [_P, _I, _P, _I, _P, _I, _I, _I, _I, _I, _I, _P],
    "lx_linear": [_P, _I, _P, _I, _I, _I, _I, _P, _I, _I, _P, _P, _P, _P, _LL, _LL, _I, _F, _P],
    "lx_linear_kn": [_P, _I, _P, _I, _I, _I, _I, _P, _I, _I, _P, _P, _P, _P, _LL, _LL, _I, _F, _P],
    "lx_predict_mlp_mask": [_P, _I, _I, _I, _P, _I, _I, _F, _I, _P, _P, _P, _P, _P, _P],
    "lx_mask_compact": [_P, _I, _I, _I, _P, _P, _P, _P],
    "lx_predict_attention_patterns": [_P, _I, _I, _I, _P, _I, _I, _I, _F, _D, _I, _P, _P, _I, _I, _P, _P, _P, _P],
    "lx_neuron_fc1": [_P, _I, _I, _I, _I, _I, _P, _P, _P, _P, _P, _P, _I, _F, _I, _P, _I, _P, _P, _P],
    "lx_neuron_fc2": [_P, _I, _I, _I, _I, _I, _I, _P, _P, _P, _P, _P, _P, _I, _F, _P, _I, _P, _P, _P],
    "lx_neuron_fc2_dgrad": [_P, _I, _I, _I, _I, _I, _P, _P, _P, _P, _P, _I, _P, _P, _I, _P, _P, _P],
    "lx_pack_active_rows": [_P, _I, _I, _I, _I, _P, _P, _P, _P],
    "lx_pack_active_rows2": [_P, _P, _I, _I, _I, _I, _P, _P, _P, _P, _P],
    "lx_lm_head_ce_nseg": [_I],
    "lx_lm_head_ce": [_P, _I, _I, _I, _P, _I, _P, _F, _P, _I, _P, _P, _P, _P, _P],
    "lx_neuron_fc1_dgrad": [_P, _I, _I, _I, _I, _I, _I, _P, _P, _P, _P, _P, _I, _P, _I, _P, _P],
    "lx_rowproj": [_P, _I, _I, _I, _I, _P, _LL, _LL, _I, _F, _P, _P, _I, _P, _I, _P, _P],
    "lx_rowproj_ws_bytes": [_I, _I, _I, _I],
    "lx_rowproj_packed": [_P, _I, _I, _I, _I, _P, _I, _I, _I, _F, _P, _P, _I, _P, _I, _P, _I, _P],
    "lx_rowproj_packed_seg": [_P, _I, _LL, _I, _I, _P, _LL, _I, _I, _I, _F, _P, _I, _I, _P, _I, _I, _I, _P],
    "lx_pack_params": [_P, _I, _P],
    "lx_colgrad_group_ws_floats": [_P, _I, _I, _I],
    "lx_colgrad_group": [_P, _I, _I, _I, _P, _P],
    "lx_bsattn_fwd_tc": [_P, _I, _I, _I, _I, _I, _P, _I, _P, _I, _F, _P, _I, _P, _P],
    "lx_bsattn_bwd_tc": [_P, _I, _I, _P, _P, _I, _I, _I, _I, _I, _P, _I, _P, _I, _F, _P, _P, _P, _P, _P],
    "lx_debug_set_attn_trace": [_P],
    "lx_adapter_ws_floats": [_I, _I],
    "lx_adapter_fwd": [_P, _I, _I, _I, _I, _P, _P, _P, _P, _P, _P, _I, _P, _I, _P],
    "lx_adapter_bwd": [_P, _I, _P, _I, _I, _I, _I, _P, _P, _P, _P, _P, _I, _P, _F, _P, _P, _P, _P, _P],
    "lx_layernorm_fwd": [_P, _P, _P, _I, _I, _P, _P, _F, _P, _I, _P, _P, _I, _I, _P, _P],
    "lx_cross_entropy": [_P, _I, _I, _P, _F, _P, _P, _P],
    "lx_adam_step": [_P, _P, _P, _P, _LL, _D, _D, _D, _D, _I, _P],
    "lx_layernorm_bwd": [_P, _I, _P, _P, _P, _P, _I, _I, _P, _P, _P],
    "lx_exact_mass_smem": [_I, _I],
    "lx_exact_block_mass": [_P, _P, _I, _I, _I, _I, _I, _I, _P, _P],
    "lx_select_by_coverage": [_P, _I, _I, _I, _P, _P, _I, _D, _I, _P, _P],
    "lx_block_importance": [_P, _I, _I, _I, _I, _I, _P, _P],
    "lx_filter_neuron_blocks": [_P, _I, _I, _D, _P, _P],
    "lx_block_activity": [_P, _I, _I, _I, _I, _P, _P],
    "lx_weighted_bce": [_P, _I, _I, _I, _P, _F, _P, _I, _P, _P],
}
RESTYPES = {"lx_last_error": C.c_char_p, "lx_colgrad_group_ws_floats": _LL, "lx_rowproj_ws_bytes": _LL, "lx_exact_mass_smem": C.c_size_t,
            "lx_adapter_ws_floats": _LL}



class ColgradProblem(C.Structure):
    """lx_colgrad_problem (include/sparseft_b200.h)."""

    _fields_ = [("p", _P), ("ldp", _I), ("x", _P), ("ldx", _I), ("ncols", _I), ("r", _I), ("scale", _F), ("pos", _P),
                ("blk", _I), ("g", _P), ("g_sq", _LL), ("g_sc", _LL)]


class PackSegment(C.Structure):
    """lx_pack_segment (include/sparseft_b200.h)."""

    _fields_ = [("src", _P), ("src_sr", _LL), ("src_sc", _LL), ("rows", _I), ("cols", _I), ("dst", _P), ("dst_sr", _LL),
                ("dst_sc", _LL), ("lo_off", _LL), ("scale", _F), ("pad_", _I)]


_ERRORS = {1: E.ShapeError, 2: E.LayoutError, 3: E.MaskError, 4: E.PatternError, 5: E.CudaError, 6: E.UnsupportedError}

_lib = None


def lib() -> C.CDLL:
    """Load (once) and return the extension; raises if it was not built."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise E.CudaError(
                f"{LIB_PATH.name} not built: run `python -m paper_2510_15964_b200.build` (no CPU fallback exists)"
            )
        handle = C.CDLL(str(LIB_PATH))
        for name, argt in SIGNATURES.items():
            if not hasattr(handle, name):
                continue  # tests/test_abi_symbols.py asserts the full set is exported
            fn = getattr(handle, name)
            fn.argtypes = argt
            fn.restype = RESTYPES.get(name, _I)
        _lib = handle
    return _lib


_NON_STATUS = ("lx_abi_version", "lx_device_sm_count", "lx_gemm_set_cta_pair", "lx_exact_mass_smem", "lx_adapter_ws_floats",
               "lx_lm_head_ce_nseg")


# Kernel-time probe (bench.py's roofline): when a dict {symbol: list}, every call of a listed symbol is
# bracketed by CUDA events on the current stream (the stream the call launches on) and the event pair is
# appended to its list. Eager steps only; never set during CUDA-graph capture.
PROBE: dict | None = None


def call(name: str, *args) -> int:
    """Invoke an entry point; map a nonzero return code to the reference's exception type."""
    if PROBE is not None and name in PROBE:
        import torch

        ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
        ev[0].record()
        rc = getattr(lib(), name)(*args)
        ev[1].record()
        PROBE[name].append(ev)
    else:
        rc = getattr(lib(), name)(*args)
    if isinstance(rc, int) and rc != 0 and name not in _NON_STATUS:
        msg = lib().lx_last_error().decode(errors="replace")
        raise _ERRORS.get(rc, E.CudaError)(f"{name}: {msg}")
    return rc


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None -> NULL)."""
    return None if t is None else t.data_ptr()


def stream_handle(device=None) -> int:
    import torch

    return torch.cuda.current_stream(device).cuda_stream
