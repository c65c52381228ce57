"""compute-sanitizer targets: the smoke iteration (memcheck) and a single
engine-v2 convolution launch (racecheck / synccheck), small shapes so the
instrumented runs finish in minutes.

    compute-sanitizer --tool memcheck python tools/sanitize_smoke.py smoke
    compute-sanitizer --tool racecheck python tools/sanitize_smoke.py tc2
"""

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def tc2_once():
    import numpy as np
    import torch

    from paper_1412_6249_b200 import _native

    lib = _native.lib()
    n, c, h, w, k, r = 2, 64, 28, 28, 96, 3
    x = torch.randn(n, c, h, w, device="cuda")
    wt = torch.randn(k, c, r, r, device="cuda")
    b = torch.randn(k, device="cuda")
    y = torch.empty(n, k, h, w, device="cuda")
    ws = torch.empty(64 << 18, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    lib("bf_conv2d_fwd", x.data_ptr(), wt.data_ptr(), b.data_ptr(), y.data_ptr(), n, c, h, w, k,
        r, r, h, w, 1, 1, ws.data_ptr(), ws.numel() * 4, st)
    torch.cuda.synchronize()
    ref = torch.nn.functional.conv2d(x.double(), wt.double(), b.double(), padding=1)
    err = float((y.double() - ref).abs().max() / ref.abs().max())
    print(f"tc2 conv forward 2x64x28x28 -> 96 3x3: max scaled err {err:.2e}")
    assert np.isfinite(err) and err < 1e-4


if __name__ == "__main__":
    if sys.argv[1:] == ["tc2"]:
        tc2_once()
    else:
        import __graft_entry__

        __graft_entry__.smoke()
