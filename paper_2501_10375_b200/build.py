"""Build libdaop_b200.so in-tree with nvcc for sm_100a (no GPU needed).

    python paper_2501_10375_b200/build.py        # or __graft_entry__.build()

(run by path: importing the package loads the library this script builds)

Every ``csrc/*.cu`` is compiled with ``-gencode arch=compute_100a,code=sm_100a``
only (``-arch=sm_100a`` would also emit compute_100 PTX, which ptxas rejects
for tcgen05) and linked into one shared library next to this file.  The
build is incremental on source / header mtimes.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OBJ = ROOT / "build" / "obj"
LIB = PKG / "libdaop_b200.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + [
    "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC,-O3,-Wall,-Wno-unused-function",
    "-Xptxas", "-O3",
    f"-I{ROOT / 'include'}",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; the CUDA 12.9 toolkit is required to build")


def _headers():
    return list(CSRC.glob("*.cuh")) + list((ROOT / "include").glob("*.h"))


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build(verbose: bool = False, extra_flags=None) -> Path:
    srcs = sorted(CSRC.glob("*.cu"))
    OBJ.mkdir(parents=True, exist_ok=True)
    hdrs = _headers()
    flags = NVCC_FLAGS + list(extra_flags or [])
    exe = nvcc()

    def compile_one(src: Path):
        obj = OBJ / (src.stem + ".o")
        if not _stale(obj, [src] + hdrs + [Path(__file__)]):
            return obj, None
        cmd = [exe, *flags, "-c", str(src), "-o", str(obj)]
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            return obj, f"{src.name}:\n{r.stdout}\n{r.stderr}"
        if verbose and r.stderr.strip():
            print(r.stderr, file=sys.stderr)
        return obj, None

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        results = list(ex.map(compile_one, srcs))
    errors = [e for _, e in results if e]
    if errors:
        raise RuntimeError("nvcc failed:\n" + "\n".join(errors))
    objs = [o for o, _ in results]
    if _stale(LIB, objs):
        cmd = [exe, *ARCH, "-shared", "-o", str(LIB), *map(str, objs),
               "-Xcompiler", "-fPIC", "-lpthread"]
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
