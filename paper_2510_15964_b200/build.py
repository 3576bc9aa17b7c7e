"""Build the in-tree CUDA extension `libsparseft_b200.so` for sm_100a.

    python -m paper_2510_15964_b200.build            # all translation units

The library is plain C-ABI (include/sparseft_b200.h), loaded with ctypes by
paper_2510_15964_b200/_abi.py. Built in-tree so it travels to the GPU box.
"""

from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OBJ = Path(os.environ.get("LX_BUILD_DIR", PKG / "build"))
LIB = Path(os.environ.get("LX_LIB_OUT", PKG / "libsparseft_b200.so"))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC,-O2", "-Xptxas", "-v,-warn-spills",
    f"-I{ROOT / 'include'}", f"-I{CSRC}",
    *os.environ.get("LX_NVCC_EXTRA", "").split(),
]


def sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu"))


def _compile(src: Path) -> tuple[Path, str]:
    obj = OBJ / (src.stem + ".o")
    deps = [src, *CSRC.glob("*.cuh"), ROOT / "include" / "sparseft_b200.h"]
    if obj.exists() and obj.stat().st_mtime > max(p.stat().st_mtime for p in deps):
        return obj, ""
    cmd = [NVCC, *FLAGS, "-c", str(src), "-o", str(obj)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src.name}:\n{r.stderr}")
    return obj, r.stderr


def build(verbose: bool = False) -> Path:
    OBJ.mkdir(exist_ok=True)
    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        results = list(ex.map(_compile, sources()))
    if verbose:
        for _, log in results:
            if log:
                print(log, file=sys.stderr)
    objs = [o for o, _ in results]
    if not LIB.exists() or LIB.stat().st_mtime < max(o.stat().st_mtime for o in objs):
        cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC", *map(str, objs),
               "-o", str(LIB), "-cudart", "static"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
