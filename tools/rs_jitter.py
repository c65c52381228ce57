"""Per-iteration timing of the drop-in run_sequence path (replay cache +
PrefetchFeed), to find where occasional slow runs lose their time.

    python tools/rs_jitter.py [--reps 6] [--iters 30]

For every repetition: device ms per iteration (events recorded by the
before_iteration hook on the current stream) and host ms per iteration.
"""

import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1412_6249_b200 import SyntheticFeed, TensorStore, init_params, run_sequence  # noqa: E402
from paper_1412_6249_b200.exchange import build_rank_sequence  # noqa: E402
from paper_1412_6249_b200.executor import PrefetchFeed  # noqa: E402
from paper_1412_6249_b200.nets import googlenet  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=6)
    ap.add_argument("--iters", type=int, default=30)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    net = googlenet(batch=128, lr=0.01)
    store = TensorStore("cuda:0")
    seq, _ = build_rank_sequence(net, 1, 0, store)
    init_params(net, store, 7, seq.layout)
    feed = SyntheticFeed.for_net(net, 7, spread=0.0)
    x, lab = feed.batch_for(0, 0)
    xname, lname = seq.layout.data_names[0], seq.layout.label_names[0]
    store.set(xname, x)
    store.set(lname, lab)
    x_pin = torch.from_numpy(x).pin_memory()
    l_pin = torch.from_numpy(lab).pin_memory()
    pf = PrefetchFeed(lambda it: {xname: x_pin, lname: l_pin}, "cuda:0")
    for rep in range(a.reps + 1):
        n = 4 if rep == 0 else a.iters
        pf.iterations = n
        evs, host = [], []

        def before(it, st):
            ev = torch.cuda.Event(enable_timing=True)
            ev.record()
            evs.append(ev)
            host.append(time.perf_counter())
            pf(it, st)

        run_sequence(seq, store, before_iteration=before, iterations=n, trace=False)
        end = torch.cuda.Event(enable_timing=True)
        end.record()
        host.append(time.perf_counter())
        end.synchronize()
        if rep == 0:
            continue
        evs.append(end)
        dev = np.array([evs[i].elapsed_time(evs[i + 1]) for i in range(n)])
        hms = np.diff(np.array(host)) * 1e3
        tot = evs[0].elapsed_time(end)
        print(f"rep {rep}: {tot:8.1f} ms = {128 * n / tot * 1e3:7.0f} img/s | device/iter "
              f"median {np.median(dev):.2f} max {dev.max():.2f} (it {int(dev.argmax())}) | "
              f"host/iter median {np.median(hms):.2f} max {hms.max():.2f} (it {int(hms.argmax())})")
        slow = [(i, round(float(d), 2), round(float(h), 2)) for i, (d, h) in enumerate(zip(dev, hms))
                if d > 1.15 * np.median(dev)]
        if slow:
            print("   slow iterations (it, device ms, host ms):", slow)


if __name__ == "__main__":
    main()
