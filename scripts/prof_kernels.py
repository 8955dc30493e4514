#!/usr/bin/env python
"""Run one libboris kernel case (for ncu --set full capture of a single launch).

    python scripts/prof_kernels.py --case aos32|aos64|soa64|fusedarr|grid|deposit|sort
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
import paper_2104_04579_b200 as lb  # noqa: E402
from paper_2104_04579_b200.ensemble import AosEnsemble, SoaEnsemble  # noqa: E402


def grid64(prec):
    dt = torch.float32 if prec == lb.BORIS_FP32 else torch.float64
    g, L = 64, 1.5 * synth.LAMBDA0
    comps = [(torch.randn((g, g, g), device="cuda", dtype=torch.float64) * 80 * synth.E_UNIT)
             .to(dt) for _ in range(6)]
    h = lb.boris_field_create_grid(0, prec, g, g, g, [-L / 2] * 3, [L / g] * 3,
                                   *(c.data_ptr() for c in comps))
    return h, comps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", required=True)
    ap.add_argument("--n", type=int, default=10_000_000)
    ap.add_argument("--steps", type=int, default=1, help="grid case: steps per push")
    a = ap.parse_args()
    n = a.n
    w = synth.config("C2", n=n)
    prec = lb.BORIS_FP64 if a.case in ("aos64", "soa64") else lb.BORIS_FP32
    cls = AosEnsemble if a.case.startswith("aos") else SoaEnsemble
    ens = cls(n, prec, w.types, w.light_velocity)
    ens.fill(w.generate(0, n, device="cuda"))
    ens.wrap()
    sp = torch.cuda.current_stream().cuda_stream
    if a.case in ("aos32", "aos64", "soa64"):
        for _ in range(3):
            lb.boris_push(ens.handle, ens.field, w.dt, 1, sp)
    elif a.case == "fusedarr":
        for _ in range(2):
            lb.boris_push(ens.handle, ens.field, w.dt, 100, sp)
    elif a.case in ("grid", "deposit", "sort"):
        h, comps = grid64(prec)
        lb.boris_ensemble_sort_by_cell(ens.handle, h, sp)
        if a.case == "grid":
            for _ in range(2):
                lb.boris_push(ens.handle, h, w.dt, a.steps, sp)
        elif a.case == "deposit":
            J = [torch.zeros((64, 64, 64), device="cuda") for _ in range(3)]
            for _ in range(2):
                lb.boris_deposit_current(ens.handle, h, w.dt, *(j.data_ptr() for j in J), sp)
        else:
            lb.boris_ensemble_sort_by_cell(ens.handle, h, sp)
        torch.cuda.synchronize()
        lb.boris_field_destroy(h)
    torch.cuda.synchronize()
    ens.close()


if __name__ == "__main__":
    main()
