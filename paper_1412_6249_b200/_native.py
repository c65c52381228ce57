"""ctypes binding of the in-tree sm_100a library (lib/libpurine_b200.so).

The library exposes the C ABI declared in ``include/purine_b200.h``.  There
is no fallback: if the shared object is missing or fails to load, every
compute kind raises `KernelError` naming the problem, so a GPU run can never
silently degrade to CPU arithmetic.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

from .kinds import KernelError

LIB_PATH = Path(__file__).resolve().parent / "lib" / "libpurine_b200.so"
if os.environ.get("PURINE_B200_LIB"):  # A/B builds of the same library (tools/)
    LIB_PATH = Path(os.environ["PURINE_B200_LIB"]).resolve()

_p = C.c_void_p
_f = C.c_float
_i = C.c_int
_l = C.c_int64

# name -> argtypes (all return int unless listed in _RESTYPE)
_SIGS = {
    "bf_version": [],
    "bf_last_error": [],
    "bf_sm_count": [_i],
    "bf_has_tcgen05": [],
    "bf_launch_count": [],
    "bf_set_gemm_engine": [_i],
    "bf_set_sm_reserve": [_i],
    "bf_set_device": [_i],
    "bf_delay_ns": [_l, _p],
    "bf_relu_fwd": [_p, _p, _l, _p],
    "bf_relu_bwd": [_p, _p, _p, _l, _p],
    "bf_relu_bwd_slice": [_p, _p, _i, _i, _p, _i, _i, _l, _p],
    "bf_relu_bwd_slice_sum": [_p, _p, _i, _i, _i, _p, _i, _i, _l, _p],
    "bf_relu_bwd_slice_x": [_p, _i, _i, _p, _i, _i, _p, _i, _i, _l, _p],
    "bf_relu_bwd_slice_sum_x": [_p, _i, _i, _p, _i, _i, _i, _p, _i, _i, _l, _p],
    "bf_sgd_update": [_p, _p, _p, _f, _l, _p],
    "bf_sgd_momentum": [_p, _p, _p, _p, _p, _f, _f, _l, _p],
    "bf_sgd_mean_update": [_p, _p, _p, _f, _i, _l, _p],
    "bf_sgd_mean_momentum": [_p, _p, _p, _p, _p, _f, _f, _i, _l, _p],
    "bf_aggregate": [_p, _i, _p, _l, _i, _p],
    "bf_copy": [_p, _i, _p, _i, _l, _p],
    "bf_check_finite": [_p, _l, _p, _p],
    "bf_check_finite_list": [_p, _p, _i, _p, _p],
    "bf_softmax_xent": [_p, _p, _p, _p, _i, _i, _p, _p],
    "bf_fc_fwd": [_p, _p, _p, _p, _i, _i, _i, _p, _l, _p],
    "bf_fc_bwd_data": [_p, _p, _p, _i, _i, _i, _p, _l, _p],
    "bf_fc_bwd_weight": [_p, _p, _p, _i, _i, _i, _p, _l, _p],
    "bf_fc_bwd_bias": [_p, _p, _i, _i, _p],
    "bf_conv1x1_fwd_group": [_p] + [_i] * 5 + [_p] * 7 + [_p, _l, _p],
    "bf_conv1x1_dgrad_group": [_i] * 5 + [_p] * 4 + [_p, _l, _p],
    "bf_conv2d_fwd": [_p, _p, _p, _p] + [_i] * 11 + [_p, _l, _p],
    "bf_conv2d_fwd_relu": [_p, _p, _p, _p, _p] + [_i] * 11 + [_p, _l, _p],
    "bf_conv2d_fwd_relu_slice": [_p, _p, _p, _p, _p, _i, _i] + [_i] * 11 + [_p, _l, _p],
    "bf_conv2d_bwd_data": [_p, _p, _p] + [_i] * 11 + [_p, _l, _p],
    "bf_conv2d_bwd_data_relu": [_p, _p, _p, _p] + [_i] * 11 + [_p, _l, _p],
    "bf_conv2d_bwd_weight": [_p, _p, _p] + [_i] * 11 + [_p, _l, _p],
    "bf_conv2d_bwd_weight_bias": [_p, _p, _p, _p] + [_i] * 11 + [_p, _l, _p],
    "bf_conv2d_bwd_bias": [_p, _p, _i, _i, _i, _p, _l, _p],
    "bf_gemm_workspace_bytes": [_i] * 12,
    "bf_maxpool_staged_ok": [_i] * 10,
    "bf_maxpool_fwd_staged": [_p, _p, _p] + [_i] * 9 + [_p],
    "bf_maxpool_bwd_x": [_p, _p, _p, _i] + [_i] * 9 + [_p],
    "bf_maxpool_bwd_staged": [_p, _p, _p] + [_i] * 9 + [_p],
    "bf_maxpool_fwd_smask": [_p, _p, _p] + [_i] * 9 + [_p],
    "bf_maxpool_bwd_smask": [_p, _p, _p, _i] + [_i] * 9 + [_p],
    "bf_maxpool_fwd": [_p, _p, _p] + [_i] * 9 + [_p],
    "bf_maxpool_bwd": [_p, _p, _p] + [_i] * 9 + [_p],
    "bf_maxpool_bwd_relu": [_p, _p, _p, _p] + [_i] * 9 + [_p],
    "bf_avgpool_fwd": [_p, _p] + [_i] * 9 + [_p],
    "bf_avgpool_bwd": [_p, _p] + [_i] * 9 + [_p],
    "bf_lrn_fwd": [_p, _p, _p, _i, _i, _i, _i, _i, _f, _f, _f, _p],
    "bf_lrn_bwd": [_p, _p, _p, _p, _p, _i, _i, _i, _i, _i, _f, _f, _f, _p],
    "bf_lrn_bwd_relu": [_p, _p, _p, _p, _p, _p, _i, _i, _i, _i, _i, _f, _f, _f, _p],
    "bf_lrn_bwd_recompute": [_p, _p, _p, _p, _i, _i, _i, _i, _i, _f, _f, _f, _p],
    "bf_concat_fwd": [_p, _p, _i, _p, _i, _i, _i, _p],
    "bf_concat_bwd": [_p, _p, _p, _i, _i, _i, _i, _p],
    "bf_nccl_unique_id": [_p],
    "bf_nccl_init": [_p, _i, _i, _p],
    "bf_nccl_destroy": [_p],
    "bf_nccl_reduce_scatter": [_p, _p, _p, _l, _p],
    "bf_nccl_all_gather": [_p, _p, _p, _l, _p],
    "bf_nccl_all_reduce": [_p, _p, _p, _l, _p],
}
_RESTYPE = {"bf_last_error": C.c_char_p, "bf_gemm_workspace_bytes": _l,
            "bf_launch_count": C.c_longlong}

_lock = threading.Lock()
_lib = None


class _Lib:
    def __init__(self, handle: C.CDLL) -> None:
        self.handle = handle
        self.fns = {}
        for name, argtypes in _SIGS.items():
            fn = getattr(handle, name)
            fn.argtypes = argtypes
            fn.restype = _RESTYPE.get(name, _i)
            self.fns[name] = fn

    def __call__(self, name: str, *args):
        rc = self.fns[name](*args)
        if rc != 0:
            msg = self.fns["bf_last_error"]().decode(errors="replace")
            raise KernelError(msg or f"{name} failed with code {rc}")
        return rc

    def raw(self, name: str):
        return self.fns[name]


def lib() -> _Lib:
    """The loaded library; raises KernelError if it was not built."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not LIB_PATH.exists():
                    raise KernelError(
                        f"CUDA kernel library not built: {LIB_PATH} is missing "
                        "(run `python -m paper_1412_6249_b200._build`); there is no CPU fallback")
                try:
                    loaded_lib = _Lib(C.CDLL(str(LIB_PATH), mode=C.RTLD_GLOBAL))
                except OSError as exc:
                    raise KernelError(f"cannot load {LIB_PATH}: {exc}") from None
                # A/B switch for the contraction engines (bf_set_gemm_engine)
                if os.environ.get("PURINE_B200_GEMM_ENGINE"):
                    loaded_lib("bf_set_gemm_engine", int(os.environ["PURINE_B200_GEMM_ENGINE"]))
                _lib = loaded_lib
    return _lib


def loaded() -> bool:
    return _lib is not None


def ptr_array(ptrs) -> C.Array:
    arr = (C.c_void_p * len(ptrs))()
    for i, p in enumerate(ptrs):
        arr[i] = p
    return arr


def int_array(vals) -> C.Array:
    arr = (C.c_int * len(vals))()
    for i, v in enumerate(vals):
        arr[i] = int(v)
    return arr
