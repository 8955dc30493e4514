#!/usr/bin/env python
"""Sorted-input deposition launches for ncu (launch 0 = warm-up, 1.. = measured).

    ncu -k regex:k_deposit -s 1 -c 1 ... python scripts/prof_deposit.py [--precision fp32]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
import paper_2104_04579_b200 as lb  # noqa: E402
from paper_2104_04579_b200.ensemble import SoaEnsemble  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=10_000_000)
ap.add_argument("--grid", type=int, default=64)
ap.add_argument("--precision", default="fp32")
ap.add_argument("--launches", type=int, default=3)
a = ap.parse_args()
prec = lb.BORIS_FP32 if a.precision == "fp32" else lb.BORIS_FP64
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
lb.boris_ensemble_sort_by_cell(ens.handle, grid, sp)
for _ in range(a.launches):
    lb.boris_deposit_current(ens.handle, grid, w.dt, *(j.data_ptr() for j in J), sp)
torch.cuda.synchronize()
