"""Build the sm_100a kernel library in-tree: csrc/*.cu -> lib/libpurine_b200.so.

Plain nvcc (no torch extension machinery): every translation unit compiles
with ``-gencode arch=compute_100a,code=sm_100a -lineinfo -O3`` in parallel,
then one ``nvcc -shared`` link against the NCCL that torch itself loads.
Run ``python -m paper_1412_6249_b200._build`` or ``__graft_entry__.build()``.
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIBDIR = PKG / "lib"
LIB = LIBDIR / "libpurine_b200.so"
INCLUDE = PKG.parent / "include"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dirs() -> tuple[Path, Path]:
    import importlib.util

    spec = importlib.util.find_spec("nvidia.nccl")
    if spec and spec.submodule_search_locations:
        root = Path(list(spec.submodule_search_locations)[0])
        if (root / "include" / "nccl.h").exists():
            return root / "include", root / "lib"
    return Path("/usr/include"), Path("/usr/lib/x86_64-linux-gnu")


def _flags(extra_inc: Path) -> list[str]:
    return ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                   "-Xptxas", "-warn-spills", "--expt-relaxed-constexpr",
                   "-I", str(INCLUDE), "-I", str(CSRC), "-I", str(extra_inc)]


def build(verbose: bool = False, force: bool = False) -> Path:
    sources = sorted(CSRC.glob("*.cu"))
    headers = sorted(CSRC.glob("*.cuh")) + sorted(INCLUDE.glob("*.h"))
    newest = max(p.stat().st_mtime for p in sources + headers + [Path(__file__)])
    if LIB.exists() and not force and LIB.stat().st_mtime >= newest:
        return LIB
    nccl_inc, nccl_lib = _nccl_dirs()
    objdir = PKG / "build"
    objdir.mkdir(exist_ok=True)
    LIBDIR.mkdir(exist_ok=True)
    flags = _flags(nccl_inc)

    def compile_one(src: Path) -> Path:
        obj = objdir / (src.stem + ".o")
        cmd = [NVCC, *flags, "-c", str(src), "-o", str(obj)]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src.name}:\n{res.stderr}")
        if verbose and res.stderr.strip():
            print(res.stderr, file=sys.stderr)
        return obj

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(compile_one, sources))
    nccl_so = nccl_lib / "libnccl.so.2"
    link = [NVCC, *ARCH, "-shared", "-o", str(LIB), *map(str, objs),
            f"-Xlinker={nccl_so}", f"-Xlinker=-rpath,{nccl_lib}"]
    res = subprocess.run(link, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(verbose=True, force="--force" in sys.argv))
