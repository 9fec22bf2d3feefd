"""In-tree build of the sm_100a C-ABI library (libcpk_b200.so).

Plain nvcc, no torch extension machinery: the library exposes only the C ABI
declared in include/cpk_b200.h, so it links against the CUDA runtime and
cuSOLVER and nothing from torch.  The .so lands next to this file under
_lib/ so it travels to the GPU box with the repo snapshot.
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
INCLUDE = ROOT / "include"
LIBDIR = PKG / "_lib"
LIB = LIBDIR / "libcpk_b200.so"
CUDA_HOME = Path(os.environ.get("CUDA_HOME", "/usr/local/cuda"))

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def sources():
    return sorted(CSRC.glob("*.cu"))


def headers():
    return sorted(CSRC.glob("*.cuh")) + sorted(INCLUDE.glob("*.h"))


def up_to_date() -> bool:
    if not LIB.exists():
        return False
    t = LIB.stat().st_mtime
    return all(p.stat().st_mtime <= t for p in sources() + headers() + [Path(__file__)])


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and up_to_date():
        return LIB
    LIBDIR.mkdir(exist_ok=True)
    objdir = LIBDIR / "obj"
    objdir.mkdir(exist_ok=True)
    nvcc = str(CUDA_HOME / "bin" / "nvcc")
    from concurrent.futures import ThreadPoolExecutor

    hdr_t = max(p.stat().st_mtime for p in headers() + [Path(__file__)])
    jobs, objs = [], []
    for src in sources():
        obj = objdir / (src.stem + ".o")
        objs.append(str(obj))
        # object cache: recompile a source only when it (or any header) changed
        if not force and obj.exists() and obj.stat().st_mtime >= max(src.stat().st_mtime, hdr_t):
            continue
        cmd = [
            nvcc, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
            "--expt-relaxed-constexpr", "-I", str(INCLUDE), "-I", str(CSRC),
            "-c", str(src), "-o", str(obj),
        ]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        jobs.append(cmd)
    with ThreadPoolExecutor(max_workers=max(1, min(len(jobs) or 1, os.cpu_count() or 1))) as ex:
        list(ex.map(lambda c: _run(c, verbose), jobs))
    link = [
        nvcc, *ARCH, "-shared", "-o", str(LIB), *objs,
        "-L", str(CUDA_HOME / "lib64"), "-lcusolver",
        "-Xlinker", f"-rpath={CUDA_HOME / 'lib64'}",
    ]
    _run(link, verbose)
    return LIB


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd), flush=True)
    res = subprocess.run(cmd, capture_output=True, text=True)
    if verbose or res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed ({res.returncode}): {' '.join(cmd[:3])} ...")


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
