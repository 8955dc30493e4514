#!/usr/bin/env python
"""Tuning experiment: HBM copy bandwidth vs size, and the C5 streaming push vs
ensemble size, back to back (the bench's regime).  One JSON line per point.

    LIBBORIS_PATH=... python scripts/exp_stream.py [--tag name] [--copy]
"""
import argparse
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402


def clocks():
    try:
        out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw",
                              "--format=csv,noheader,nounits"], capture_output=True,
                             text=True).stdout.strip()
        return out
    except Exception:
        return ""


def timed(fn, iters):
    st = torch.cuda.current_stream()
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(iters):
        fn()
    b.record(st)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", default=os.environ.get("LIBBORIS_PATH", "default"))
    ap.add_argument("--copy", action="store_true")
    ap.add_argument("--sizes", default="1e8,2e8,4e8,8e8")
    args = ap.parse_args()
    if args.copy:
        for gb in (2, 8, 32):
            n = gb * (1 << 30) // 2
            a = torch.empty(n, dtype=torch.bfloat16, device="cuda")
            b = torch.empty_like(a)
            ms = timed(lambda: b.copy_(a), 20)
            print(json.dumps({"exp": "torch_copy", "bytes_each_way": gb << 30,
                              "gbs": 2 * (gb << 30) / (ms * 1e-3) / 1e9, "clk": clocks()}),
                  flush=True)
            del a, b
            torch.cuda.empty_cache()
    import synth
    import paper_2104_04579_b200 as lb
    from paper_2104_04579_b200.ensemble import SoaEnsemble
    lb.load_library()
    for n in [int(float(s)) for s in args.sizes.split(",")]:
        w = synth.config("C5", n=n)
        ens = SoaEnsemble(n, lb.BORIS_FP32, w.types, w.light_velocity)
        for c0 in range(0, n, 1 << 24):
            ens.fill(w.generate(c0, min(1 << 24, n - c0), device="cuda"), first=c0)
        ens.wrap()
        d = torch.zeros(2, dtype=torch.float64, device="cuda")
        sp = torch.cuda.current_stream().cuda_stream
        iters = max(20, int(100 * 8e8 / n))
        ms = timed(lambda: lb.boris_push_diag(ens.handle, ens.field, w.dt, 1, d.data_ptr(), sp),
                   iters)
        print(json.dumps({"exp": "c5_stream", "tag": args.tag, "n": n, "iters": iters,
                          "ms": ms, "gbs": 80 * n / (ms * 1e-3) / 1e9, "clk": clocks()}),
              flush=True)
        ens.close()
        del ens
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
