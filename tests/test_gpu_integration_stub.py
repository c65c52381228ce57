"""INTEGRATION.md section 2 binds the C ABI with plain ctypes (no package
import): this runs that binding's calls -- the same argtypes, the same
argument order, torch device buffers -- against the CPU oracle, so the
documented stub is known to work as written."""

import ctypes as C
from pathlib import Path

import numpy as np
import pytest

import oracle as O
from gpu_util import assert_close

pytestmark = pytest.mark.gpu

LIB = Path(__file__).resolve().parent.parent / "paper_1412_6249_b200" / "lib" / "libpurine_b200.so"


def _lib():
    lib = C.CDLL(str(LIB))
    lib.bf_last_error.restype = C.c_char_p
    P, I, L = C.c_void_p, C.c_int, C.c_int64
    lib.bf_relu_fwd.argtypes = [P, P, L, P]
    lib.bf_conv2d_fwd.argtypes = [P, P, P, P] + [I] * 11 + [P, L, P]
    return lib


def _check(lib, rc):
    if rc:
        raise RuntimeError(lib.bf_last_error().decode())


def test_documented_ctypes_binding_runs():
    import torch

    lib = _lib()
    rng = np.random.default_rng(3)
    stream = torch.cuda.current_stream().cuda_stream
    ws = torch.empty(256 << 20, device="cuda")  # GEMM workspace, as in the stub

    x = rng.standard_normal((2, 3, 16, 16)).astype(np.float32)
    xd = torch.from_numpy(x).cuda()
    y = torch.empty_like(xd)
    _check(lib, lib.bf_relu_fwd(xd.data_ptr(), y.data_ptr(), xd.numel(), stream))
    torch.cuda.synchronize()
    assert np.array_equal(y.cpu().numpy(), O.relu_forward(x))

    w = (rng.standard_normal((8, 3, 3, 3)) / np.sqrt(27)).astype(np.float32)
    b = rng.standard_normal(8).astype(np.float32)
    wd, bd = torch.from_numpy(w).cuda(), torch.from_numpy(b).cuda()
    s, p = 1, 1
    n, c, h, wdt = x.shape
    k, _, r, ss = w.shape
    ho, wo = (h + 2 * p - r) // s + 1, (wdt + 2 * p - ss) // s + 1
    out = torch.empty((n, k, ho, wo), device="cuda")
    _check(lib, lib.bf_conv2d_fwd(xd.data_ptr(), wd.data_ptr(), bd.data_ptr(), out.data_ptr(),
                                  n, c, h, wdt, k, r, ss, ho, wo, s, p, ws.data_ptr(),
                                  ws.numel() * 4, stream))
    torch.cuda.synchronize()
    want = O.conv2d_forward(x, w, b, s, p)
    assert_close(out.cpu().numpy(), want, rtol=1e-4, atol=1e-5 * max(1.0, float(np.abs(want).max())),
                 what="conv via the documented binding")
