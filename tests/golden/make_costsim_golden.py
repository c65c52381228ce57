"""Golden schedules for the cost simulator, produced by the REFERENCE
`biflow.costsim.simulate` (run in the build container, where /root/reference
exists; the GPU box only reads the committed costsim.json).

For every reference-built graph sequence in graphs.json (cfg1, the 2-peer DP
MLP fused / split) the reference simulates 2
iterations under a fixed cost model: per-kind constant costs, copies by
latency + bytes / bandwidth.  Output: makespan and the full trace (name,
lane thread, start ns, end ns, iteration).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_costsim_golden.py
"""

import json
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")

from biflow import costsim as rc  # noqa: E402
from biflow.graph import graph_from_json as ref_from_json  # noqa: E402

KIND_COST_US = {"conv2d_forward": 40, "conv2d_backward": 90, "conv2d_backward_data": 45,
                "conv2d_backward_weight": 50, "conv2d_backward_bias": 5, "fc_forward": 12,
                "fc_backward": 30, "fc_backward_data": 14, "fc_backward_weight": 15,
                "fc_backward_bias": 2, "relu_forward": 3, "relu_backward": 4,
                "flatten_forward": 1, "flatten_backward": 1, "softmax_xent": 6,
                "sgd_update": 2, "aggregate": 3, "swap": 0, "maxpool_forward": 7,
                "maxpool_backward": 9}


def model():
    return rc.CostModel(kind_costs={k: v * 1e-6 for k, v in KIND_COST_US.items()},
                        bandwidth=25e9, latency=2e-6)


def main():
    graphs = json.loads((HERE / "graphs.json").read_text())
    out = {"kind_cost_us": KIND_COST_US, "bandwidth": 25e9, "latency": 2e-6, "cases": {}}
    for tag in ("cfg1", "mlp_dp2_fused", "mlp_dp2_split"):
        gs = [ref_from_json(g) for g in graphs[tag]["graphs"]]
        seq = rc.GraphSequence(gs, iterations=2)
        rep = rc.simulate(seq, model(), images_per_iteration=16)
        out["cases"][tag] = {
            "makespan": rep.makespan, "throughput": rep.throughput,
            "trace": [[r.name, r.lane.thread, r.start, r.end, r.iteration] for r in rep.trace]}
    (HERE / "costsim.json").write_text(json.dumps(out, sort_keys=True) + "\n")


if __name__ == "__main__":
    main()
