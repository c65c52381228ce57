"""Where the e2e (host batch in, loss out) step loses time against the
device-resident step: times K captured GoogLeNet steps with / without the
per-step prefetch of the pinned batch and the per-step async loss read.

    python tools/e2e_probe.py [--steps 20]
"""

import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_1412_6249_b200 import SyntheticFeed, TensorStore, init_params  # noqa: E402
from paper_1412_6249_b200.exchange import build_rank_sequence  # noqa: E402
from paper_1412_6249_b200.executor import CapturedSequence  # noqa: E402
from paper_1412_6249_b200.nets import googlenet  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    net = googlenet(batch=128, lr=0.01)
    store = TensorStore("cuda:0")
    seq, _ = build_rank_sequence(net, 1, 0, store)
    init_params(net, store, 7, seq.layout)
    x, lab = SyntheticFeed.for_net(net, 7, spread=0.0).batch_for(0, 0)
    xn, ln = seq.layout.data_names[0], seq.layout.label_names[0]
    store.set(xn, x)
    store.set(ln, lab)
    loss = seq.layout.loss_names[0]
    exe = CapturedSequence(seq, store)
    exe.prepare()
    xp = torch.from_numpy(x).pin_memory()
    lp = torch.from_numpy(lab).pin_memory()
    for _ in range(3):
        exe.step()
    torch.cuda.synchronize()

    def run(prefetch, read):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        if prefetch:
            exe.prefetch({xn: xp, ln: lp})
        reads = []
        for s in range(a.steps):
            exe.step()
            if read:
                reads.append(store.read_async(loss))
            if prefetch and s + 1 < a.steps:
                exe.prefetch({xn: xp, ln: lp})
        e1.record()
        e1.synchronize()
        for r in reads:
            r.value()
        return e0.elapsed_time(e1) / a.steps

    for prefetch, read in ((0, 0), (0, 1), (1, 0), (1, 1), (0, 0)):
        ms = run(prefetch, read)
        print(f"prefetch={prefetch} read={read}: {ms:.3f} ms/step = {128 / ms * 1e3:.0f} img/s")
    # H2D bandwidth alone
    buf = torch.empty_like(xp, device="cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        buf.copy_(xp, non_blocking=True)
    e1.record()
    e1.synchronize()
    print(f"H2D {xp.numel() * 4 / 1e6:.0f} MB: {e0.elapsed_time(e1) / 5:.3f} ms "
          f"({xp.numel() * 4 * 5 / e0.elapsed_time(e1) / 1e6:.1f} GB/s)")


if __name__ == "__main__":
    main()
