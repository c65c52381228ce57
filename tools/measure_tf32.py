"""Measure the dense TF32 tensor peak on this B200 (cuBLAS via torch.matmul,
8192^3, allow_tf32) the same way MEASURED_PEAKS.json measures bf16: best of
10 (burst) and back-to-back for ~4 s (sustained).  Writes
profiles/tf32_peak.json; bench.py divides it by 3 for the 3xTF32 roofline."""

import json
import sys
import time
from pathlib import Path

import torch

OUT = Path(__file__).resolve().parent.parent / "profiles" / "tf32_peak.json"


def main():
    torch.backends.cuda.matmul.allow_tf32 = True
    n = 8192
    a = torch.randn(n, n, device="cuda")
    b = torch.randn(n, n, device="cuda")
    for _ in range(3):
        a @ b
    torch.cuda.synchronize()
    best = 0.0
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        a @ b
        e1.record()
        e1.synchronize()
        best = max(best, 2 * n ** 3 / (e0.elapsed_time(e1) / 1e3) / 1e12)
    t0 = time.time()
    iters = 0
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    while time.time() - t0 < 4.0:
        for _ in range(10):
            a @ b
        iters += 10
        torch.cuda.synchronize()
    e1.record()
    e1.synchronize()
    sustained = 2 * n ** 3 * iters / (e0.elapsed_time(e1) / 1e3) / 1e12
    rec = {"tf32_tflops": best, "tf32_tflops_sustained": sustained,
           "how": "torch.matmul fp32 8192^3 with allow_tf32 (cuBLAS TF32 tensor cores); best of 10 "
                  "and back-to-back ~4 s", "gpu": torch.cuda.get_device_name(0),
           "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())}
    OUT.parent.mkdir(exist_ok=True)
    OUT.write_text(json.dumps(rec, indent=1) + "\n")
    print(json.dumps(rec))
    return 0


if __name__ == "__main__":
    sys.exit(main())
