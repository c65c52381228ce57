"""Build an A/B variant of the kernel library with extra -D defines.

    python tools/build_variant.py OUT.so -DTC2_EPI_WARPS=4 -DTC2_PREFETCH=0

Load it with PURINE_B200_LIB=OUT.so (paper_1412_6249_b200/_native.py).
"""

import concurrent.futures as cf
import subprocess
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_1412_6249_b200 import _build as B  # noqa: E402


def main():
    out = Path(sys.argv[1]).resolve()
    defines = sys.argv[2:]
    inc, lib = B._nccl_dirs()
    objdir = out.parent / (out.stem + "_obj")
    objdir.mkdir(parents=True, exist_ok=True)
    flags = B._flags(inc) + defines

    def one(src):
        obj = objdir / (src.stem + ".o")
        r = subprocess.run([B.NVCC, *flags, "-c", str(src), "-o", str(obj)], capture_output=True,
                           text=True)
        if r.returncode:
            raise RuntimeError(r.stderr)
        return obj

    with cf.ThreadPoolExecutor(8) as ex:
        objs = list(ex.map(one, sorted(B.CSRC.glob("*.cu"))))
    nccl = lib / "libnccl.so.2"
    r = subprocess.run([B.NVCC, *B.ARCH, "-shared", "-o", str(out), *map(str, objs),
                        f"-Xlinker={nccl}", f"-Xlinker=-rpath,{lib}"], capture_output=True, text=True)
    if r.returncode:
        raise RuntimeError(r.stderr)
    print(out)


if __name__ == "__main__":
    main()
