"""Time the staged max-pool kernels: float mask / recompute-from-x / signed mask.

    python tools/pool_mask_bench.py
"""

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_1412_6249_b200 import _native  # noqa: E402

SHAPES = [((128, 64, 112, 112), 2, 0), ((128, 192, 56, 56), 2, 0), ((128, 480, 28, 28), 2, 0),
          ((128, 256, 28, 28), 1, 1), ((128, 480, 14, 14), 1, 1), ((128, 832, 7, 7), 1, 1)]


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps * 1e3


def main():
    lib = _native.lib()
    st = torch.cuda.current_stream().cuda_stream
    for (n, c, h, w), s, p in SHAPES:
        ph, pw = -(-(h + 2 * p - 3) // s) + 1, -(-(w + 2 * p - 3) // s) + 1  # ceil mode
        x = torch.relu(torch.randn(n, c, h, w, device="cuda"))
        y = torch.empty(n, c, ph, pw, device="cuda")
        m = torch.empty_like(y)
        dy = torch.randn_like(y)
        dx = torch.empty_like(x)
        sm = torch.empty_like(y)
        a = (n, c, h, w, ph, pw, 3, s, p, st)
        r = {}
        r["fwd"] = timeit(lambda: lib("bf_maxpool_fwd_staged", x.data_ptr(), y.data_ptr(), 0, *a))
        r["fwd+mask"] = timeit(lambda: lib("bf_maxpool_fwd_staged", x.data_ptr(), y.data_ptr(),
                                           m.data_ptr(), *a))
        r["fwd+smask"] = timeit(lambda: lib("bf_maxpool_fwd_smask", x.data_ptr(), y.data_ptr(),
                                            sm.data_ptr(), *a))
        if lib.raw("bf_maxpool_staged_ok")(n, c, h, w, ph, pw, 3, s, p, 1):
            r["bwd_x relu"] = timeit(lambda: lib("bf_maxpool_bwd_x", x.data_ptr(), dy.data_ptr(),
                                                 dx.data_ptr(), 1, *a))
        if lib.raw("bf_maxpool_staged_ok")(n, c, h, w, ph, pw, 3, s, p, 2):
            r["bwd_mask"] = timeit(lambda: lib("bf_maxpool_bwd_staged", m.data_ptr(), dy.data_ptr(),
                                               dx.data_ptr(), *a))
        for rf in (0, 1):
            r[f"bwd_smask relu={rf}"] = timeit(lambda: lib("bf_maxpool_bwd_smask", sm.data_ptr(),
                                                           dy.data_ptr(), dx.data_ptr(), rf, *a))
        print(f"{(n, c, h, w)} s{s}: " + "  ".join(f"{k} {v:6.1f}us" for k, v in r.items()))


if __name__ == "__main__":
    main()
