"""Summarise ncu outputs into markdown for profiles/.

    python tools/summarize_ncu.py launches gpurun_out/launches.csv > profiles/rXX_launches.md
    python tools/summarize_ncu.py full gpurun_out/prof.ncu-rep > profiles/rXX_<kernel>.md

`launches`: per-kernel-family count / total / share of device time from a
``--metrics gpu__time_duration.sum`` CSV (cold-cache, serialised: compare
shares, not absolutes).  `full`: the headline metrics of a ``--set full``
capture (duration, DRAM bytes, pipe utilisation, occupancy, stall mix).
"""

import csv
import io
import re
import subprocess
import sys
from collections import defaultdict


def family(name: str) -> str:
    n = name.replace("<unnamed>::", "").replace("(anonymous namespace)::", "")
    n = re.sub(r"^void ", "", n)
    m = re.match(r"(?:bf::)?tc::tc_gemm_kernel<bf::(\w+), bf::(\w+), bf::(\w+), (?:\(int\))?(\d+), "
                 r"(?:\(int\))?(\d+)>", n)
    if m:
        return f"tc_gemm<{m.group(1)},{m.group(2)},{m.group(3)},BN={m.group(4)}>"
    m = re.match(r"(?:bf::)?tc(\d)::tc\d_kernel<(?:bf::)?(\w+), (?:bf::)?(\w+)(?:, (?:\(int\))?(\d+))?>", n)
    if m:
        return f"tc{m.group(1)}<{m.group(2)},{m.group(3)}{',mode=' + m.group(4) if m.group(4) else ''}>"
    n = re.sub(r"\(.*", "", n)
    n = re.sub(r"<.*", "", n)
    return n


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    data = []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                data.append((d["Kernel Name"], float(d["Metric Value"])))
    agg = defaultdict(lambda: [0, 0.0])
    for name, ns in data:
        f = family(name)
        agg[f][0] += 1
        agg[f][1] += ns
    total = sum(v[1] for v in agg.values())
    print(f"launches: {len(data)}, total device time {total / 1e6:.3f} ms\n")
    print("| kernel family | launches | total ms | share |")
    print("|---|---:|---:|---:|")
    for f, (c, ns) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| `{f}` | {c} | {ns / 1e6:.3f} | {ns / total:.1%} |")
    if len(sys.argv) > 3:  # also the N longest single launches, in launch order index
        top = sorted(enumerate(data), key=lambda kv: -kv[1][1])[:int(sys.argv[3])]
        print("\n| launch # | kernel | us |\n|---:|---|---:|")
        for i, (name, ns) in top:
            print(f"| {i} | `{family(name)}` | {ns / 1e3:.1f} |")


KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "smsp__average_warp_latency_issue_stalled_long_scoreboard",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_sleeping_per_issue_active.ratio"]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        print(f"### `{family(d.get('Kernel Name', '?'))}`\n")
        print("| metric | value |")
        print("|---|---:|")
        for k in KEYS:
            if k in d:
                print(f"| {k} | {d[k]} {u.get(k, '')} |")
        rd = float(d.get("dram__bytes_read.sum", "0").replace(",", "") or 0)
        wr = float(d.get("dram__bytes_write.sum", "0").replace(",", "") or 0)
        print(f"| traffic (read+write) | {rd + wr:.4g} {u.get('dram__bytes_read.sum', '')} |\n")


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
