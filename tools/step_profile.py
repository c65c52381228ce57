"""One captured training step bracketed by cudaProfilerStart/Stop, for ncu.

    ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
        --csv --log-file gpurun_out/step_launches.csv python tools/step_profile.py
    python tools/summarize_ncu.py launches gpurun_out/step_launches.csv

Builds exactly the bench's rank sequence (exchange-lowered GoogLeNet / NIN
iteration, batch 128), captures it, runs warm-up replays, then profiles ONE
replay: the launch list covers precisely the kernels of one timed step.
"""

import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_1412_6249_b200 import SyntheticFeed, TensorStore, init_params  # noqa: E402
from paper_1412_6249_b200.exchange import build_rank_sequence  # noqa: E402
from paper_1412_6249_b200.executor import CapturedSequence  # noqa: E402
from paper_1412_6249_b200.nets import googlenet, nin  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--net", default="googlenet", choices=["googlenet", "nin"])
    ap.add_argument("--batch", type=int, default=128)
    ap.add_argument("--warmup", type=int, default=3)
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
    exe = CapturedSequence(seq, store)
    exe.prepare()
    for _ in range(a.warmup):
        exe.step()
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    exe.step()
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print("profiled one step;", exe.launches_per_step, "library launches per step")


if __name__ == "__main__":
    main()
