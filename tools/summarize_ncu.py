"""Summarise ncu outputs into markdown for profiles/.

    python tools/summarize_ncu.py launches gpurun_out/launches.csv > profiles/rXX_launches.md
    python tools/summarize_ncu.py full gpurun_out/prof.ncu-rep > profiles/rXX_<kernel>.md

`launches`: per-kernel-family count / total / share of device time from a
``--metrics gpu__time_duration.sum`` CSV (cold-cache, serialised: compare
shares, not absolutes).  `full`: the headline metrics of a ``--set full``
capture (duration, DRAM bytes, pipe utilisation, occupancy, stall mix).
`traffic`: per-family time and DRAM bytes from a ``--metrics
gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum`` CSV of one
step (tools/step_profile.py), plus a JSON summary (argv[3]) that bench.py
reports as ``roofline.traffic``.
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


_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "usecond": 1e3,
          "us": 1e3, "msecond": 1e6, "ms": 1e6, "nsecond": 1}
# kernels of the conv / fc contraction family (the tensor-bound roofline's
# "kernel"): the implicit GEMMs plus their pack / split-K / bias side kernels
_CONTRACTION = re.compile(r"^(?:\w+::)*(tc\d?_kernel|tc\d?<|tc_gemm|pack_|splitk_|bias_\w*finish|"
                         r"simt_gemm|gemm_)")


def traffic(path, out_json=None):
    import json

    rows = list(csv.reader(open(path)))
    hdr = None
    per = defaultdict(dict)  # launch id -> metric -> value
    names = {}
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            v = float(d["Metric Value"].replace(",", "")) * _SCALE.get(d["Metric Unit"], 1)
            per[d["ID"]][d["Metric Name"]] = v
            names[d["ID"]] = d["Kernel Name"]
    agg = defaultdict(lambda: [0, 0.0, 0.0])
    for lid, m in per.items():
        f = family(names[lid])
        a = agg[f]
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0.0)
        a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    tot_t = sum(a[1] for a in agg.values())
    print(f"launches: {len(per)}, serialised device time {tot_t / 1e6:.3f} ms, DRAM "
          f"{sum(a[2] for a in agg.values()) / 1e9:.3f} GB\n")
    print("| kernel family | launches | ms | share | DRAM MB | GB/s |")
    print("|---|---:|---:|---:|---:|---:|")
    for f, (c, ns, by) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| `{f}` | {c} | {ns / 1e6:.3f} | {ns / tot_t:.1%} | {by / 1e6:.1f} | "
              f"{by / ns if ns else 0:.0f} |")
    con = [a for f, a in agg.items() if _CONTRACTION.match(f)]
    oth = [a for f, a in agg.items() if not _CONTRACTION.match(f)]
    summary = {"source": path, "launches": len(per), "serialised_ms": tot_t / 1e6,
               "contraction": {"launches": sum(a[0] for a in con),
                               "ms": sum(a[1] for a in con) / 1e6,
                               "dram_bytes": sum(a[2] for a in con)},
               "hbm_kernels": {"launches": sum(a[0] for a in oth),
                               "ms": sum(a[1] for a in oth) / 1e6,
                               "dram_bytes": sum(a[2] for a in oth)}}
    print("\n```json\n" + json.dumps(summary, indent=1) + "\n```")
    if out_json:
        with open(out_json, "w") as fh:
            json.dump(summary, fh, indent=1)


if __name__ == "__main__":
    {"launches": launches, "full": full, "traffic": traffic}[sys.argv[1]](*sys.argv[2:])
