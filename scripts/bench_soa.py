#!/usr/bin/env python
"""Single-step SoA push (C2 shapes, boris_push: 76 / 152 B): ps per particle-step and layout-implied GB/s.

    python scripts/bench_soa.py [--n 10000000]
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
import paper_2104_04579_b200 as lb  # noqa: E402
from paper_2104_04579_b200.ensemble import SoaEnsemble  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=10_000_000)
    ap.add_argument("--iters", type=int, default=20)
    a = ap.parse_args()
    st = torch.cuda.current_stream()
    for prec, name, bpp in ((lb.BORIS_FP32, "fp32", 76), (lb.BORIS_FP64, "fp64", 152)):
        w = synth.config("C2", n=a.n)
        ens = SoaEnsemble(a.n, prec, w.types, w.light_velocity)
        ens.fill(w.generate(0, a.n, device="cuda"))
        ens.wrap()
        for _ in range(3):
            lb.boris_push(ens.handle, ens.field, w.dt, 1, st.cuda_stream)
        torch.cuda.synchronize()
        ts = []
        for _ in range(a.iters):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            lb.boris_push(ens.handle, ens.field, w.dt, 1, st.cuda_stream)
            e1.record(st)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = statistics.mean(ts)
        print(json.dumps({"exp": "soa_push", "precision": name, "n": a.n, "ms": ms,
                          "ps_per_particle_step": ms * 1e9 / a.n,
                          "gbs": bpp * a.n / ms / 1e6}), flush=True)
        ens.close()


if __name__ == "__main__":
    main()
