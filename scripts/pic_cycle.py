#!/usr/bin/env python
"""The particle half of a PIC cycle on one B200 (field
interpolation -> push -> current deposition; the Maxwell solve is out of scope):
every step gathers E, B from a grid (CIC) inside the push, then deposits J; the
ensemble is re-sorted by cell every `--sort-every` steps (L233-236).

    python scripts/pic_cycle.py [--n 10000000] [--grid 64] [--steps 50] [--sort-every 10]
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
    ap.add_argument("--n", type=int, default=10_000_000)
    ap.add_argument("--grid", type=int, default=64)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--sort-every", type=int, default=10)
    ap.add_argument("--precision", default="fp32")
    ap.add_argument("--fused", action="store_true",
                    help="push + deposit in one call (boris_push_deposit)")
    a = ap.parse_args()
    prec = lb.BORIS_FP32 if a.precision == "fp32" else lb.BORIS_FP64
    dt_ = torch.float32 if prec == lb.BORIS_FP32 else torch.float64
    g = a.grid
    L = 1.5 * synth.LAMBDA0
    gen = torch.Generator(device="cuda").manual_seed(5)
    comps = [(torch.randn((g, g, g), generator=gen, device="cuda", dtype=torch.float64)
              * 80 * synth.E_UNIT).to(dt_) for _ in range(6)]
    grid = lb.boris_field_create_grid(0, prec, g, g, g, [-L / 2] * 3, [L / g] * 3,
                                      *(c.data_ptr() for c in comps))
    J = [torch.zeros((g, g, g), device="cuda", dtype=dt_) for _ in range(3)]
    w = synth.config("C5", n=a.n)
    ens = SoaEnsemble(a.n, prec, w.types, w.light_velocity, with_fields=False)
    ens.fill(w.generate(0, a.n, device="cuda"))
    ens.wrap()
    st = torch.cuda.current_stream()
    sp = st.cuda_stream
    diag = torch.zeros(2, dtype=torch.float64, device="cuda")
    ev = {k: [] for k in ("sort", "push", "deposit")}

    def timed(kind, fn):
        a0 = torch.cuda.Event(enable_timing=True)
        a1 = torch.cuda.Event(enable_timing=True)
        a0.record(st)
        fn()
        a1.record(st)
        ev[kind].append((a0, a1))

    for step in range(a.steps + 2):  # 2 warm-up steps
        if step % a.sort_every == 0:
            timed("sort", lambda: lb.boris_ensemble_sort_by_cell(ens.handle, grid, sp))
        if a.fused:
            timed("push", lambda: lb.boris_push_deposit(ens.handle, grid, w.dt,
                                                        *(j.data_ptr() for j in J),
                                                        diag.data_ptr(), sp))
        else:
            timed("push", lambda: lb.boris_push_diag(ens.handle, grid, w.dt, 1, diag.data_ptr(),
                                                     sp))
            timed("deposit", lambda: lb.boris_deposit_current(ens.handle, grid, w.dt,
                                                              *(j.data_ptr() for j in J), sp))
        if step == 1:
            torch.cuda.synchronize()
            ev = {k: [] for k in ev}
    torch.cuda.synchronize()
    ms = {k: sum(a0.elapsed_time(a1) for a0, a1 in v) for k, v in ev.items()}
    total = sum(ms.values())
    out = {"exp": "pic_particle_cycle", "precision": a.precision, "fused": a.fused,
           "n": a.n, "cells": g ** 3,
           "steps": a.steps, "sort_every": a.sort_every,
           "ms_per_step": {k: v / a.steps for k, v in ms.items()},
           "ps_per_particle_step": total * 1e9 / (a.n * a.steps),
           "kinetic_energy_erg": diag[0].item(), "count": diag[1].item()}
    print(json.dumps(out), flush=True)
    ens.close()
    lb.boris_field_destroy(grid)


if __name__ == "__main__":
    main()
