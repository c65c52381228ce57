"""Critical path of one traced, branch-concurrent training step.

    python tools/critical_path.py [--net googlenet] [--batch 128] [--top 40]

Replays the bench's captured step with per-operator CUDA events (the timed
schedule: fusion plan, branch streams), then walks back from the operator
that ends last: at each operator the blocking predecessor is the producer of
one of its inputs (or the same-graph operator waited on) with the latest end
time.  Prints the chain with each operator's device time and the idle gap
before it, plus per-kind totals on the chain -- the operators whose speed-up
shortens the step.  (Event timing serialises nothing but adds ~2 us per
operator; absolute times are a little above the untraced step's.)
"""

import argparse
import sys
from collections import defaultdict
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_1412_6249_b200 import SyntheticFeed, TensorStore, init_params  # noqa: E402
from paper_1412_6249_b200.dispatcher import _env_lane_cap, _plan  # noqa: E402
from paper_1412_6249_b200.exchange import build_rank_sequence  # noqa: E402
from paper_1412_6249_b200.executor import CapturedSequence  # noqa: E402
from paper_1412_6249_b200.nets import googlenet, nin  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--net", default="googlenet", choices=["googlenet", "nin"])
    ap.add_argument("--batch", type=int, default=128)
    ap.add_argument("--top", type=int, default=60)
    ap.add_argument("--tail", type=int, default=25, help="print the chain's last N operators")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    net = (googlenet if a.net == "googlenet" else nin)(batch=a.batch, lr=0.01)
    store = TensorStore("cuda:0")
    seq, _ = build_rank_sequence(net, 1, 0, store)
    init_params(net, store, 7, seq.layout)
    feed = SyntheticFeed.for_net(net, 7, spread=0.0)
    x, lab = feed.batch_for(0, 0)
    store.set(seq.layout.data_names[0], x)
    store.set(seq.layout.label_names[0], lab)
    exe = CapturedSequence(seq, store, trace=True)
    exe.prepare()
    for _ in range(4):
        par = exe.parity
        exe.step()
    torch.cuda.synchronize()
    iv = [(op, s0, s1) for gi, op, s0, s1 in exe.op_intervals_ns(par) if gi == 0]
    g = seq.graphs[0]
    plan = _plan(g, _env_lane_cap())
    span = {}
    for op, s0, s1 in iv:
        span[op.name] = (s0, s1)
    oid_of = {op.name: oid for oid, op in g.operators.items()}

    def preds(oid):
        out = set()
        for t in g.operators[oid].inputs:
            p = g.producer_of(t)
            if p is not None:
                out.add(p)
        out.update(plan.waits.get(oid, []))
        return out

    end_op = max(iv, key=lambda r: r[2])[0]
    chain = []
    cur = oid_of[end_op.name]
    while cur is not None:
        op = g.operators[cur]
        s0, s1 = span[op.name]
        best, best_end = None, -1
        for p in preds(cur):
            pn = g.operators[p].name
            if pn in span and span[pn][1] <= s1 and span[pn][1] > best_end:
                best, best_end = p, span[pn][1]
        chain.append((op, s0, s1, s0 - best_end if best is not None else 0))
        cur = best
    chain.reverse()
    total = chain[-1][2] - chain[0][1]
    print(f"step (graph 0) {max(r[2] for r in iv) / 1e6:.3f} ms; critical chain "
          f"{len(chain)} ops, {total / 1e6:.3f} ms, busy "
          f"{sum(s1 - s0 for _, s0, s1, _ in chain) / 1e6:.3f} ms")
    by_kind = defaultdict(float)
    for op, s0, s1, gap in chain:
        by_kind[op.kind] += (s1 - s0) / 1e6
    for k, v in sorted(by_kind.items(), key=lambda kv: -kv[1]):
        print(f"  {k:26s} {v:7.3f} ms")
    print(f"\nlast {a.tail} operators of the chain (start ms, device ms, gap us):")
    for op, s0, s1, gap in chain[-a.tail:]:
        print(f"  {op.name:34s} {op.kind:24s} {s0 / 1e6:7.3f} {(s1 - s0) / 1e6:7.3f}  gap {gap / 1e3:7.1f}")
    # what else runs during the chain's last operators
    t_end = chain[-1][2]
    t0 = chain[-min(a.tail, len(chain))][1]
    others = sorted((r for r in iv if r[2] > t0 and r[0].name not in {c[0].name for c in chain}),
                    key=lambda r: r[1])
    print(f"\noff-chain operators overlapping the last {(t_end - t0) / 1e6:.3f} ms:")
    for op, s0, s1 in others[:40]:
        print(f"  {op.name:34s} {op.kind:24s} {s0 / 1e6:7.3f} {(s1 - s0) / 1e6:7.3f}")
    rows = sorted(chain, key=lambda r: -(r[2] - r[1]))[:a.top]
    print("\nlongest operators on the chain (device ms, idle gap before it us):")
    for op, s0, s1, gap in rows:
        fz = ",".join(sorted(plan.fusion.get(oid_of[op.name], {}).keys()))
        print(f"  {op.name:34s} {op.kind:24s} {(s1 - s0) / 1e6:7.3f}  gap {gap / 1e3:7.1f}  {fz}")


if __name__ == "__main__":
    main()
