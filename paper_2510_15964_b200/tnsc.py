"""The `.tnsc` tensor file format of the reference (sf/containers.py), read and written
byte-for-byte compatibly so traces and predictor files move between the two.

    offset 0   b"TNSC"
    offset 4   u32 LE format version (1)
    offset 8   u32 LE length L of the header
    offset 12  L bytes of JSON, keys sorted: {"tensors": [{"dtype", "layout", "name", "shape"}, ...]}
    then       each payload in header order; "layout": "col" payloads are Fortran-ordered

Element types: float32, float64, int64. Payloads are memory-mapped on read (one
copy per tensor, no whole-file read), and torch tensors — including device
tensors — are accepted on write.
"""

from __future__ import annotations

import json
import mmap
import struct
from pathlib import Path

import numpy as np

TNSC_MAGIC = b"TNSC"
TNSC_VERSION = 1
_PREFIX = struct.Struct("<4sII")
_ELEM = {"float32": np.dtype(np.float32), "float64": np.dtype(np.float64), "int64": np.dtype(np.int64)}


class ContainerError(ValueError):
    """Malformed or unsupported file (the reference's ContainerError, sf/containers.py:24)."""


def _as_numpy(value) -> np.ndarray:
    if hasattr(value, "detach"):  # torch tensor, possibly on the GPU
        return value.detach().cpu().numpy()
    return np.asarray(value)


def save_tensors(path, tensors: dict, column_major=frozenset()) -> None:
    """Write `tensors` (name -> array) in insertion order; names in `column_major` are stored
    Fortran-ordered (sf/containers.py:28-49)."""
    missing = sorted(set(column_major).difference(tensors))
    if missing:
        raise ContainerError(f"column_major names not present: {missing}")
    entries, blobs = [], []
    for name, value in tensors.items():
        a = _as_numpy(value)
        if a.dtype.name not in _ELEM:
            raise ContainerError(f"unsupported dtype {a.dtype.name} for tensor {name!r}")
        fortran = name in column_major
        entries.append({"name": name, "dtype": a.dtype.name, "shape": [int(n) for n in a.shape],
                        "layout": "col" if fortran else "row"})
        blobs.append(a.tobytes(order="F" if fortran else "C"))
    head = json.dumps({"tensors": entries}, sort_keys=True).encode("utf-8")
    with open(path, "wb") as f:
        f.write(_PREFIX.pack(TNSC_MAGIC, TNSC_VERSION, len(head)))
        f.write(head)
        for b in blobs:
            f.write(b)


def load_tensors(path) -> tuple[dict[str, np.ndarray], set[str]]:
    """Read a file; returns (name -> array, names stored column-major) (sf/containers.py:52-78)."""
    with open(path, "rb") as f:
        try:
            buf = mmap.mmap(f.fileno(), 0, access=mmap.ACCESS_READ)
        except ValueError:  # empty file
            raise ContainerError(f"{path}: bad magic") from None
    with buf:
        if len(buf) < _PREFIX.size or buf[:4] != TNSC_MAGIC:
            raise ContainerError(f"{path}: bad magic")
        _, version, head_len = _PREFIX.unpack_from(buf, 0)
        if version != TNSC_VERSION:
            raise ContainerError(f"{path}: unsupported version {version}")
        pos = _PREFIX.size + head_len
        spec = json.loads(bytes(buf[_PREFIX.size : pos]).decode("utf-8"))
        out: dict[str, np.ndarray] = {}
        fortran_names: set[str] = set()
        for e in spec["tensors"]:
            elem = _ELEM.get(e["dtype"])
            if elem is None:
                raise ContainerError(f"{path}: unsupported dtype {e['dtype']}")
            shape = tuple(e["shape"])
            count = int(np.prod(shape, dtype=np.int64))
            if pos + count * elem.itemsize > len(buf):
                raise ContainerError(f"{path}: truncated payload for {e['name']!r}")
            flat = np.frombuffer(buf, dtype=elem, count=count, offset=pos).copy()
            pos += count * elem.itemsize
            if e["layout"] == "col":
                fortran_names.add(e["name"])
                out[e["name"]] = np.asfortranarray(flat.reshape(shape, order="F"))
            else:
                out[e["name"]] = flat.reshape(shape)
        return out, fortran_names
