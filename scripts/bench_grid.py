#!/usr/bin/env python
"""Grid-field gather push: unsorted vs sorted by cell, and the
cost of the periodic sort itself.  One JSON line per measurement.

    python scripts/bench_grid.py [--n 10000000] [--grid 64] [--steps 100]
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


def timed(fn, iters, warmup=1):
    st = torch.cuda.current_stream()
    for _ in range(warmup):
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
    ap.add_argument("--steps", type=int, default=100)
    a = ap.parse_args()
    for prec_name, prec in (("fp32", lb.BORIS_FP32), ("fp64", lb.BORIS_FP64)):
        dt = torch.float32 if prec == lb.BORIS_FP32 else torch.float64
        g = a.grid
        L = 1.5 * synth.LAMBDA0
        gen = torch.Generator(device="cuda").manual_seed(3)
        comps = [(torch.randn((g, g, g), generator=gen, device="cuda", dtype=torch.float64)
                  * 80 * synth.E_UNIT).to(dt).contiguous() for _ in range(6)]
        grid = lb.boris_field_create_grid(0, prec, g, g, g, [-L / 2] * 3, [L / g] * 3,
                                          *(c.data_ptr() for c in comps))
        w = synth.config("C2", n=a.n)
        w.dt = synth.T0 / 1e4
        ens = SoaEnsemble(a.n, prec, w.types, w.light_velocity, with_fields=False)
        state0 = w.generate(0, a.n, device="cuda")
        ens.fill(state0)
        ens.wrap()
        sp = torch.cuda.current_stream().cuda_stream
        for order in ("unsorted", "sorted"):
            if order == "sorted":
                # random order: refill the unsorted state before each timed sort
                ts = []
                for _ in range(4):
                    ens.fill(state0)
                    ts.append(timed(lambda: lb.boris_ensemble_sort_by_cell(ens.handle, grid, sp),
                                    1, warmup=0))
                ms_sort = statistics.median(ts[1:])
                # already sorted (the periodic re-sort of a PIC loop is close to this)
                ms_pre = timed(lambda: lb.boris_ensemble_sort_by_cell(ens.handle, grid, sp), 3)
                for kind, ms_k in (("random", ms_sort), ("presorted", ms_pre)):
                    print(json.dumps({"exp": "sort_by_cell", "precision": prec_name,
                                      "input": kind, "n": a.n, "cells": g ** 3, "ms": ms_k,
                                      "ns_per_particle": ms_k * 1e6 / a.n}), flush=True)
            for steps in (1, a.steps):
                ms = timed(lambda: lb.boris_push(ens.handle, grid, w.dt, steps, sp), 5)
                print(json.dumps({"exp": "grid_push", "precision": prec_name, "order": order,
                                  "n": a.n, "cells": g ** 3, "steps": steps, "ms": ms,
                                  "ps_per_particle_step": ms * 1e9 / (a.n * steps)}),
                      flush=True)
        ens.close()
        lb.boris_field_destroy(grid)


if __name__ == "__main__":
    main()
