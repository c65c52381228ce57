"""Raw tensor files: the reference's dataset format (ops.py:464-492).

Layout, little-endian: uint32 rank (1..4), rank x uint32 dims (each >= 1),
then prod(dims) float32 values in C order.  Host-side I/O for the CLI's
``"data": {"kind": "file"}`` feed; batches are copied to the device by the
store like synthetic ones.
"""

from __future__ import annotations

import struct

import numpy as np

from .kinds import KernelError

MAX_RANK = 4


def write_tensor_file(path: str, array) -> None:
    arr = np.ascontiguousarray(array, dtype="<f4")
    if not 1 <= arr.ndim <= MAX_RANK or min(arr.shape) < 1:
        raise KernelError(f"tensor file: unsupported shape {arr.shape}")
    with open(path, "wb") as fh:
        fh.write(struct.pack(f"<{1 + arr.ndim}I", arr.ndim, *arr.shape))
        fh.write(arr.tobytes())


def read_tensor_file(path: str) -> np.ndarray:
    with open(path, "rb") as fh:
        raw = fh.read()
    if len(raw) < 4:
        raise KernelError(f"tensor file {path!r}: truncated header")
    rank = struct.unpack_from("<I", raw)[0]
    if not 1 <= rank <= MAX_RANK or len(raw) < 4 * (1 + rank):
        raise KernelError(f"tensor file {path!r}: bad rank {rank}")
    dims = struct.unpack_from(f"<{rank}I", raw, 4)
    if min(dims) < 1:
        raise KernelError(f"tensor file {path!r}: bad dim {min(dims)}")
    want = 4 * int(np.prod(dims))
    body = memoryview(raw)[4 * (1 + rank):]
    if len(body) != want:
        raise KernelError(f"tensor file {path!r}: payload is {len(body)} bytes, expected {want}")
    return np.frombuffer(body, dtype="<f4").reshape(dims).astype(np.float32)
