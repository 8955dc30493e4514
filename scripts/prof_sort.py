#!/usr/bin/env python
"""Sort launches for ncu: one random-order sort, then `--presorted` re-sorts of the sorted
ensemble (the periodic re-sort of a PIC loop is close to this).

    ncu --metrics gpu__time_duration.sum --csv ... python scripts/prof_sort.py
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
ap.add_argument("--presorted", type=int, default=2)
a = ap.parse_args()
g = a.grid
L = 1.5 * synth.LAMBDA0
comps = [torch.zeros((g, g, g), device="cuda") for _ in range(6)]
grid = lb.boris_field_create_grid(0, lb.BORIS_FP32, g, g, g, [-L / 2] * 3, [L / g] * 3,
                                  *(c.data_ptr() for c in comps))
w = synth.config("C2", n=a.n)
ens = SoaEnsemble(a.n, lb.BORIS_FP32, w.types, w.light_velocity, with_fields=False)
ens.fill(w.generate(0, a.n, device="cuda"))
ens.wrap()
sp = torch.cuda.current_stream().cuda_stream
for _ in range(1 + a.presorted):
    lb.boris_ensemble_sort_by_cell(ens.handle, grid, sp)
torch.cuda.synchronize()
