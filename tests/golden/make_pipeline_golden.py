"""Golden fixtures for the model-parallel pipeline, from the REFERENCE.

Run in the build container (where /root/reference exists):

    python tests/golden/make_pipeline_golden.py

Imports ``biflow`` from /root/reference/pkg/src (read-only, no bytecode) and
records, for build_model_parallel_pipeline (builders.py:650-776) run by the
reference dispatcher in serial mode (BIFLOW_LANES=1):
  * ``mlp3x3``: the reference tests' 3-stage fc pipeline over 3 replicas
    (test_builders.py:268-308, seed 21),
  * ``conv2x4``: config 1's conv(32,k5,p2)+relu | fc10 split into 2 stages
    over 4 micro-batches of 16 (seed 7),
their graph JSON, serial-mode dispatch order, parameters, inputs and every
replica's output -> pipeline.json / pipeline.npz.  The staircase makespans
of the reference simulator with unit stage costs are recorded too.
"""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import biflow  # noqa: E402
from biflow import builders as rb  # noqa: E402
from biflow import costsim as rc  # noqa: E402
from biflow import ops as rops  # noqa: E402
from biflow.dispatcher import run_sequence as ref_run_sequence  # noqa: E402
from biflow.graph import graph_to_json as ref_graph_to_json  # noqa: E402


CASES = {
    "mlp3x3": dict(
        net=rb.NetSpec((8,), (rb.LayerSpec("fc", 8), rb.LayerSpec("fc", 8), rb.LayerSpec("fc", 4)),
                       batch=4),
        stages=((0, 1), (1, 2), (2, 3)), replicas=3, seed=21),
    "conv2x4": dict(
        net=rb.NetSpec((3, 32, 32), (rb.LayerSpec("conv", 32, 5, 1, 2), rb.LayerSpec("relu"),
                                     rb.LayerSpec("fc", 10)), batch=16, lr=1e-3),
        stages=((0, 2), (2, 3)), replicas=4, seed=7),
}


def main() -> None:
    graphs, arrays = {}, {}
    for tag, c in CASES.items():
        plan = rb.ParallelPlan(scheme="model", replicas=c["replicas"],
                               stages=tuple(rb.Stage(s, biflow.Location("local", k))
                                            for k, s in enumerate(c["stages"])))
        seq = rb.build_model_parallel_pipeline(c["net"], plan)
        store = rops.TensorStore()
        rb.init_params(c["net"], store, c["seed"], seq.layout)
        rb.fill_tokens(store, seq)
        rng = np.random.default_rng(c["seed"])
        shape = seq.graphs[0].tensor_named("x_r0").shape
        for r in range(c["replicas"]):
            x = rng.standard_normal(shape).astype(np.float32)
            store.set(f"x_r{r}", x)
            arrays[f"{tag}_x_r{r}"] = x
        reps = ref_run_sequence(seq, store, max_workers=1)
        order = [[t.name for t in sorted(rep.trace, key=lambda t: t.start)] for rep in reps]
        for name in seq.layout.canonical_params:
            arrays[f"{tag}_{name}"] = store.array(name)
        for name in seq.layout.output_names:
            arrays[f"{tag}_{name}"] = store.array(name)
        timed = rb.build_model_parallel_pipeline(c["net"], plan)
        compute = [op for op in timed.graphs[0].operators.values()
                   if op.kind not in ("copy", "gate")]
        for op in compute:
            op.attrs["delay_s"] = 1.0
        makespan = rc.simulate(timed, rc.CostModel(kind_costs={})).makespan
        graphs[tag] = {"graphs": [ref_graph_to_json(g) for g in seq.graphs], "serial": order,
                       "layout": {"data": list(seq.layout.data_names),
                                  "tokens": list(seq.layout.token_names),
                                  "outputs": list(seq.layout.output_names),
                                  "params": list(seq.layout.canonical_params)},
                       "unit_cost_makespan": makespan}
    np.savez_compressed(HERE / "pipeline.npz", **arrays)
    (HERE / "pipeline.json").write_text(json.dumps(graphs, sort_keys=True) + "\n")
    print("wrote pipeline.json / pipeline.npz:", {k: v["unit_cost_makespan"]
                                                  for k, v in graphs.items()})


if __name__ == "__main__":
    os.environ["BIFLOW_LANES"] = "1"
    main()
