"""Non-finite detection on the GPU path (the reference's `_finite` check,
ops.py:61-64, reported first-error-wins by dispatcher.py:344-346).

The device check is one pass per graph over its sink tensors into a sticky
flag; when it fires the first operator (serial order) holding a non-finite
output is named exactly as the reference names it."""

import numpy as np
import pytest

from paper_1412_6249_b200 import (DispatchError, SyntheticFeed, TensorStore, build_sgd_iteration,
                                  feeder, init_params, run, run_sequence)
from paper_1412_6249_b200.executor import CapturedSequence
from paper_1412_6249_b200.nets import conv_relu_fc

pytestmark = pytest.mark.gpu

WANT = "operator 'conv1' failed: conv2d_forward: non-finite value in output"


def _setup(poison: str | None):
    net = conv_relu_fc()
    seq = build_sgd_iteration(net)
    store = TensorStore("cuda:0")
    init_params(net, store, 7, seq.layout)
    feeder(SyntheticFeed.for_net(net, 7, spread=0.0), seq.layout)(0, store)
    if poison:
        w = store.array(poison).copy()
        w.reshape(-1)[3] = np.nan
        store.set(poison, w)
    return net, seq, store


@pytest.mark.parametrize("mode", ["sinks", "all"])
def test_run_names_first_nonfinite_operator(monkeypatch, mode):
    monkeypatch.setenv("PURINE_B200_CHECK_FINITE", mode)
    _, seq, store = _setup("w1")
    with pytest.raises(DispatchError) as ei:
        run(seq.graphs[0], store)
    assert str(ei.value) == WANT


def test_run_sequence_untraced_raises_at_end(monkeypatch):
    _, seq, store = _setup("w1")
    with pytest.raises(DispatchError, match="non-finite value in output"):
        run_sequence(seq, store, iterations=1, trace=False)


def test_finite_run_does_not_raise_and_flag_stays_clear():
    _, seq, store = _setup(None)
    run_sequence(seq, store, iterations=2)
    assert store.has_finite_flag() and not store.finite_flag_set()


def test_check_disabled(monkeypatch):
    monkeypatch.setenv("PURINE_B200_CHECK_FINITE", "0")
    _, seq, store = _setup("w1")
    run(seq.graphs[0], store)  # no check: trains on NaNs like a plain numpy loop would
    assert not np.isfinite(store.array("a1")).all()  # the conv output
    assert not np.isfinite(store.array("w1_new")).all()


def test_captured_sequence_raises():
    _, seq, store = _setup(None)
    exe = CapturedSequence(seq, store)
    exe.prepare()
    exe.step()
    exe.sync()  # finite so far
    w = store.array("w1").copy()
    w.reshape(-1)[0] = np.inf
    store.set("w1", w)
    with pytest.raises(DispatchError) as ei:
        for _ in range(4):  # the pinned flag mirror is read a step late
            exe.step()
        exe.sync()
    assert str(ei.value) == WANT
