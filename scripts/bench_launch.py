#!/usr/bin/env python
"""Launch-bound pushes: small ensembles, many launches (the per-launch cost of the
C ABI + kernel parameter block).  One JSON line per case.

    python scripts/bench_launch.py [--n 4096] [--launches 2000]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
import paper_2104_04579_b200 as lb  # noqa: E402
from paper_2104_04579_b200.ensemble import SoaEnsemble  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--launches", type=int, default=2000)
    a = ap.parse_args()
    st = torch.cuda.current_stream()
    for cfg, steps in (("C2", 1), ("C4", 1), ("C4", 10)):
        w = synth.config(cfg, n=a.n)
        ens = SoaEnsemble(a.n, lb.BORIS_FP32, w.types, w.light_velocity,
                          with_fields=w.field_kind == "arrays")
        ens.fill(w.generate(0, a.n, device="cuda"))
        ens.wrap()
        if w.field_kind == "arrays":
            f, own = ens.field, False
        else:
            pw = w.plane_wave
            f, own = lb.boris_field_create_plane_wave(pw["E0"], pw["k_hat"], pw["e_hat"],
                                                      pw["omega"], pw["k"], pw["phase0"]), True
        for _ in range(50):
            lb.boris_push(ens.handle, f, w.dt, steps, st.cuda_stream)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(a.launches):
            lb.boris_push(ens.handle, f, w.dt, steps, st.cuda_stream)
        e1.record(st)
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / a.launches
        print(json.dumps({"exp": "launch", "cfg": cfg, "n": a.n, "steps": steps,
                          "us_per_push": us}), flush=True)
        if own:
            lb.boris_field_destroy(f)
        ens.close()


if __name__ == "__main__":
    main()
