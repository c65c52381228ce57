"""Host-side logic without a GPU: the non-finite watch list of the dispatcher
plan, the lane-threaded oracle executor used by the CPU reference arm, and
bench.py's multi-rank launch guard."""

import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from oracle.serial import run_graph_lanes, run_graph_serial
from paper_1412_6249_b200 import (DispatchError, Location, ParallelPlan, SyntheticFeed,
                                  build_data_parallel, build_sgd_iteration, feeder, init_params)
from paper_1412_6249_b200.dispatcher import _Plan
from paper_1412_6249_b200.nets import cifar_convnet, conv_relu_fc

ROOT = Path(__file__).resolve().parent.parent


def test_finite_watch_sinks_and_all(monkeypatch):
    seq = build_sgd_iteration(conv_relu_fc())
    g = seq.graphs[0]
    plan = _Plan(g, 8)
    # the loss, every updated parameter and the unused input gradient: nothing
    # in the graph reads them
    assert sorted(plan.finite_watch) == sorted(["loss", "w3_new", "b3_new", "dx", "w1_new",
                                                "b1_new"])
    monkeypatch.setenv("PURINE_B200_CHECK_FINITE", "all")
    full = _Plan(g, 8).finite_watch
    assert set(plan.finite_watch) < set(full)
    assert "a1" in full or any(n.startswith("a") for n in full)
    monkeypatch.setenv("PURINE_B200_CHECK_FINITE", "0")
    assert _Plan(g, 8).finite_watch == []
    assert _Plan(seq.graphs[1], 8).finite_watch == []  # the swap graph computes nothing
    monkeypatch.setenv("PURINE_B200_CHECK_FINITE", "bogus")
    with pytest.raises(DispatchError):
        _Plan(g, 8)


class _S(dict):
    def set(self, name, arr):
        self[name] = np.array(arr, dtype=np.float32, copy=True)


def test_lane_threaded_oracle_equals_serial():
    """The CPU reference arm's executor (reference multi-worker mode) computes
    exactly what the serial executor computes: every operator's inputs are
    fixed by the graph and the aggregate sums in rank order."""
    net = cifar_convnet(batch=4, lr=1e-3)
    plan = ParallelPlan("data", peers=(Location("local", 0), Location("local", 1)),
                        server=Location("local", 2))
    seq = build_data_parallel(net, plan)
    feed = feeder(SyntheticFeed.for_net(net, 3, peers=2, spread=0.0), seq.layout)
    a, b = _S(), _S()
    for st, runner in ((a, run_graph_serial), (b, run_graph_lanes)):
        init_params(net, st, 3, seq.layout)
        for it in range(2):
            feed(it, st)
            for g in seq.graphs:
                runner(g, st)
    assert set(a) == set(b)
    for k in a:
        assert np.array_equal(a[k].view(np.uint32), b[k].view(np.uint32)), k


def test_bench_multi_gpu_guard_fails_loudly():
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    env.pop("WORLD_SIZE", None)
    res = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--steps", "1"],
                         capture_output=True, text=True, env=env, timeout=300)
    assert res.returncode == 2, res.stderr[-2000:]
    assert "needs 2 visible CUDA devices" in json.loads(res.stdout.strip().splitlines()[-1])["error"]
