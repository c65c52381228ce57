"""Helpers for the GPU parity tests: run one operator through the product
boundary (graph -> dispatcher -> OpKindSpec.execute -> C ABI) on cuda:0."""

import numpy as np

from paper_1412_6249_b200 import BiGraph, Location, TensorStore, run

LOC = Location("local", 0)

# the NS tolerance for floating-point results (BASELINE.json north_star)
RTOL, ATOL = 1e-4, 1e-5


def run_op(kind, ins: dict, outs: dict, attrs=None, store=None):
    """ins: name -> ndarray; outs: name -> shape.  Returns {out name: ndarray}."""
    g = BiGraph()
    in_ids = [g.add_tensor(n, a.shape, LOC) for n, a in ins.items()]
    out_ids = [g.add_tensor(n, s, LOC) for n, s in outs.items()]
    g.add_operator("op", kind, in_ids, out_ids, LOC, attrs=dict(attrs or {}))
    store = store or TensorStore("cuda:0")
    for n, a in ins.items():
        store.set(n, a)
    run(g, store)
    return {n: store.array(n) for n in outs}


def assert_close(got, want, rtol=RTOL, atol=ATOL, what=""):
    got, want = np.asarray(got), np.asarray(want)
    assert got.shape == want.shape, (what, got.shape, want.shape)
    bad = ~np.isclose(got, want, rtol=rtol, atol=atol)
    if bad.any():
        i = np.argwhere(bad)[0]
        raise AssertionError(f"{what}: {bad.sum()} / {bad.size} elements off, first at {tuple(i)}: "
                             f"got {got[tuple(i)]!r} want {want[tuple(i)]!r}; max abs err "
                             f"{np.abs(got - want).max():.3e}")


def assert_bitwise(got, want, what=""):
    got, want = np.ascontiguousarray(got, np.float32), np.ascontiguousarray(want, np.float32)
    assert got.shape == want.shape, (what, got.shape, want.shape)
    diff = got.view(np.uint32) != want.view(np.uint32)
    assert not diff.any(), f"{what}: {diff.sum()} elements differ bitwise"
