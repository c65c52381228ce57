"""Device-resident tensor store.

Drop-in for the reference's `Tensor` / `TensorStore` / `swap`
(`pkg/src/biflow/ops.py:79-157`): names are the cross-graph identity, a
name's shape is fixed once set, `swap` exchanges two storage handles in
O(1) without touching any element.

B200 layout: every tensor lives in HBM of the store's CUDA device as a
float32 buffer allocated once (kernels write their outputs in place into the
preallocated buffer instead of allocating per operator, ops.py:116-130).
`set` copies host data in; `array` copies a snapshot out; `tensor` hands out
the device buffer itself.  Flatten outputs are zero-cost aliases of their
input buffer (a reshape, as in ops.py:379-391).
"""

from __future__ import annotations

from dataclasses import dataclass

import functools
import itertools

import numpy as np
import torch

from .kinds import MAX_RANK, KernelError

__all__ = ["Tensor", "TensorStore", "swap", "check_shape"]


def check_shape(shape) -> tuple[int, ...]:
    dims = tuple(shape)
    if not (1 <= len(dims) <= MAX_RANK) or any(not isinstance(d, int) or d < 1 for d in dims):
        raise KernelError(f"invalid tensor shape {dims!r}")
    return dims


def _default_device() -> torch.device:
    if torch.cuda.is_available():
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


@dataclass
class Tensor:
    """A shaped float32 buffer; ``data`` is the (device) storage handle."""

    shape: tuple[int, ...]
    data: torch.Tensor

    @classmethod
    def from_array(cls, array, device=None) -> "Tensor":
        t = _as_f32_tensor(array, device or _default_device())
        return cls(check_shape(tuple(int(d) for d in t.shape)), t.contiguous())

    @property
    def ptr(self) -> int:
        return self.data.data_ptr()

    @property
    def numel(self) -> int:
        return self.data.numel()


def swap(a: Tensor, b: Tensor) -> tuple[Tensor, Tensor]:
    """Exchange the storage handles of two equal-shaped tensors (ops.py:93-102)."""
    if a.shape != b.shape:
        raise KernelError(f"swap: shape mismatch {a.shape} vs {b.shape}")
    a.data, b.data = b.data, a.data
    return a, b


def _as_f32_tensor(array, device) -> torch.Tensor:
    if isinstance(array, torch.Tensor):
        return array.detach().to(device=device, dtype=torch.float32)
    arr = np.ascontiguousarray(array, dtype=np.float32)
    return torch.from_numpy(arr).to(device)


class PendingRead:
    """Result of `TensorStore.read_async`."""

    def __init__(self, host, event, shape) -> None:
        self._host, self._event, self._shape = host, event, shape

    def value(self) -> np.ndarray:
        self._event.synchronize()
        return self._host.numpy().reshape(self._shape)


@functools.lru_cache(maxsize=65536)
def _pair_code(a: str, b: str) -> int:
    """Deterministic 64-bit code of a swapped name pair (the swap signature)."""
    import hashlib

    return int.from_bytes(hashlib.blake2b(f"{a}\0{b}".encode(), digest_size=8).digest(), "little")


class TensorStore:
    """Named device buffers shared by every graph of a run."""

    _serials = itertools.count(1)

    def __init__(self, device=None) -> None:
        self.device = torch.device(device) if device is not None else _default_device()
        self._tensors: dict[str, Tensor] = {}
        self._alias_of: dict[str, str] = {}
        # buffer-binding signature (the dispatcher's replay cache key): a
        # process-unique store serial, an epoch bumped whenever a name is
        # (re)bound to memory, and an order-free accumulator of swaps (a swap
        # graph is an involution: swapping a pair twice restores the value)
        self._serial = next(TensorStore._serials)
        self._epoch = 0
        self._swap_sig = 0

    def binding_sig(self) -> tuple[int, int, int]:
        return (self._serial, self._epoch, self._swap_sig)

    # -- reference API ------------------------------------------------------

    def set(self, name: str, array) -> Tensor:
        """Write ``array`` (numpy or torch, any device) into ``name``'s buffer.

        An existing buffer is overwritten in place on the current stream
        (pinned host tensors copy asynchronously); a new name gets a fresh
        buffer owned by the store."""
        cur = self._tensors.get(name)
        if cur is not None and isinstance(array, torch.Tensor) and array.dtype == torch.float32:
            shape = check_shape(tuple(int(d) for d in array.shape))
            if cur.shape != shape:
                raise KernelError(f"store: shape mismatch writing {name!r}: {shape} vs existing "
                                  f"{cur.shape}")
            src = array.reshape(cur.data.shape)
            cur.data.copy_(src, non_blocking=src.device.type == "cpu" and src.is_pinned())
            return cur
        if cur is not None and not isinstance(array, torch.Tensor):
            host = np.ascontiguousarray(array, dtype=np.float32)
            shape = check_shape(tuple(int(d) for d in host.shape))
            if cur.shape != shape:
                raise KernelError(f"store: shape mismatch writing {name!r}: {shape} vs existing "
                                  f"{cur.shape}")
            cur.data.copy_(torch.from_numpy(host).reshape(cur.data.shape))
            return cur
        src = _as_f32_tensor(array, self.device)
        shape = check_shape(tuple(int(d) for d in src.shape))
        if cur is None:
            t = Tensor(shape, src.contiguous().clone())  # the store owns its buffers
            self._tensors[name] = t
            self._epoch += 1
            return t
        if cur.shape != shape:
            raise KernelError(f"store: shape mismatch writing {name!r}: {shape} vs existing {cur.shape}")
        cur.data.copy_(src.reshape(cur.data.shape))
        return cur

    def get(self, name: str) -> Tensor:
        t = self._tensors.get(name)
        if t is None:
            raise KernelError(f"store: no tensor named {name!r}")
        return t

    def array(self, name: str) -> np.ndarray:
        """Host snapshot (synchronises with the work that produced it)."""
        return self.get(name).data.detach().cpu().numpy().reshape(self.get(name).shape)

    def read_async(self, name: str) -> "PendingRead":
        """Device->host copy of ``name`` enqueued on the current stream into
        pinned memory; `.value()` waits for it.  Lets a training loop read
        every step's loss without stalling the host between steps."""
        t = self.get(name)
        host = torch.empty(t.data.shape, dtype=torch.float32, pin_memory=True)
        host.copy_(t.data, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        return PendingRead(host, ev, t.shape)

    def has(self, name: str) -> bool:
        return name in self._tensors

    def names(self) -> list[str]:
        return sorted(self._tensors)

    def swap(self, name_a: str, name_b: str) -> None:
        swap(self.get(name_a), self.get(name_b))
        lo, hi = sorted((name_a, name_b))
        self._swap_sig ^= _pair_code(lo, hi)

    def remove(self, name: str) -> None:
        self._tensors.pop(name, None)
        self._alias_of.pop(name, None)
        self._epoch += 1

    def __contains__(self, name: str) -> bool:
        return name in self._tensors

    def __len__(self) -> int:
        return len(self._tensors)

    # -- device-side extensions --------------------------------------------
    def finite_flag(self) -> torch.Tensor:
        """Sticky device int32 set by the dispatcher's per-graph non-finite check."""
        f = getattr(self, "_finite", None)
        if f is None:
            f = torch.zeros(1, dtype=torch.int32, device=self.device)
            self._finite = f
        return f

    def has_finite_flag(self) -> bool:
        return getattr(self, "_finite", None) is not None

    def finite_flag_set(self) -> bool:
        return bool(int(self.finite_flag().item()))

    def reset_finite_flag(self) -> None:
        self.finite_flag().zero_()


    def tensor(self, name: str) -> torch.Tensor:
        return self.get(name).data

    def ensure(self, name: str, shape: tuple[int, ...]) -> Tensor:
        """Preallocate an output buffer (uninitialised) if it does not exist."""
        cur = self._tensors.get(name)
        shape = check_shape(tuple(shape))
        if cur is None:
            cur = Tensor(shape, torch.empty(shape, dtype=torch.float32, device=self.device))
            self._tensors[name] = cur
            self._epoch += 1
        elif cur.shape != shape:
            raise KernelError(f"store: shape mismatch for {name!r}: {shape} vs existing {cur.shape}")
        return cur

    def alias(self, name: str, src: str, shape: tuple[int, ...]) -> Tensor:
        """Make ``name`` a reshaped view of ``src``'s current buffer."""
        base = self.get(src)
        shape = check_shape(tuple(shape))
        view = base.data.view(shape)
        cur = self._tensors.get(name)
        if cur is None:
            cur = Tensor(shape, view)
            self._tensors[name] = cur
        else:
            if cur.shape != shape:
                raise KernelError(f"store: shape mismatch aliasing {name!r}")
            cur.data = view
        self._alias_of[name] = src
        self._epoch += 1
        return cur

    def place(self, name: str, view: torch.Tensor) -> Tensor:
        """Bind ``name`` to a caller-laid-out view (e.g. a slice of a flat
        parameter/gradient arena).  Existing contents are copied in."""
        shape = check_shape(tuple(int(d) for d in view.shape))
        cur = self._tensors.get(name)
        if cur is not None:
            if cur.shape != shape:
                raise KernelError(f"store: shape mismatch placing {name!r}")
            view.copy_(cur.data)
            cur.data = view
            self._epoch += 1
            return cur
        t = Tensor(shape, view)
        self._tensors[name] = t
        self._epoch += 1
        return t

    def is_alias_of(self, name: str, src: str) -> bool:
        if self._alias_of.get(name) != src or name not in self._tensors or src not in self._tensors:
            return False
        return self._tensors[name].data.data_ptr() == self._tensors[src].data.data_ptr()
