#!/usr/bin/env python
"""Current deposition throughput: unsorted vs sorted by cell.

    python scripts/bench_deposit.py [--n 10000000] [--grid 64]
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


def timed(fn, iters=5):
    st = torch.cuda.current_stream()
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=10_000_000)
    ap.add_argument("--grid", type=int, default=64)
    a = ap.parse_args()
    for prec_name, prec in (("fp32", lb.BORIS_FP32), ("fp64", lb.BORIS_FP64)):
        dt = torch.float32 if prec == lb.BORIS_FP32 else torch.float64
        g = a.grid
        L = 1.5 * synth.LAMBDA0
        comps = [torch.zeros((g, g, g), device="cuda", dtype=dt) for _ in range(6)]
        grid = lb.boris_field_create_grid(0, prec, g, g, g, [-L / 2] * 3, [L / g] * 3,
                                          *(c.data_ptr() for c in comps))
        J = [torch.zeros((g, g, g), device="cuda", dtype=dt) for _ in range(3)]
        w = synth.config("C2", n=a.n)
        ens = SoaEnsemble(a.n, prec, w.types, w.light_velocity, with_fields=False)
        ens.fill(w.generate(0, a.n, device="cuda"))
        ens.wrap()
        sp = torch.cuda.current_stream().cuda_stream
        for order in ("unsorted", "sorted"):
            if order == "sorted":
                lb.boris_ensemble_sort_by_cell(ens.handle, grid, sp)
            ms = timed(lambda: lb.boris_deposit_current(ens.handle, grid, w.dt,
                                                        *(j.data_ptr() for j in J), sp))
            print(json.dumps({"exp": "deposit_current", "precision": prec_name, "order": order,
                              "n": a.n, "cells": g ** 3, "ms": ms,
                              "ps_per_particle": ms * 1e9 / a.n}), flush=True)
        ens.close()
        lb.boris_field_destroy(grid)


if __name__ == "__main__":
    main()
