"""Build the oracle's C restatement (TEST / BASELINE INFRASTRUCTURE ONLY):
oracle/cpu_moe.c -> oracle/_build/liboracle_cpu.so with gcc (OpenMP, the
host's vector ISA).  Called by __graft_entry__.build(); the .so is
git-ignored and travels to the GPU box with the repo snapshot."""

from __future__ import annotations

import shutil
import subprocess
from pathlib import Path

HERE = Path(__file__).resolve().parent
OUT = HERE / "_build" / "liboracle_cpu.so"


def build() -> Path:
    src = HERE / "cpu_moe.c"
    if OUT.exists() and OUT.stat().st_mtime >= src.stat().st_mtime:
        return OUT
    OUT.parent.mkdir(exist_ok=True)
    cc = shutil.which("gcc") or "gcc"
    # x86-64-v4 (AVX-512) rather than -march=native: the build container and
    # the GPU box are different hosts
    cmd = [cc, "-O3", "-march=x86-64-v4", "-fopenmp", "-shared", "-fPIC", str(src), "-o",
           str(OUT), "-lm"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"oracle C build failed:\n{r.stderr}")
    return OUT


if __name__ == "__main__":
    print(build())
