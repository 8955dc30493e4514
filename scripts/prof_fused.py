#!/usr/bin/env python
"""Launch one fused analytic push (for ncu): C4 plane wave (default), m-dipole, or the
C3 crossed uniform field.

    python scripts/prof_fused.py [--field plane_wave|mdipole|uniform] [--precision fp32|fp64]
                                 [--n 10000000] [--steps 100] [--reps 3]
"""
import argparse
import math
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
    ap.add_argument("--field", default="plane_wave")
    ap.add_argument("--precision", default="fp32")
    ap.add_argument("--n", type=int, default=10_000_000)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    w = synth.config("C3" if a.field == "uniform" else "C4", n=a.n)
    prec = lb.BORIS_FP32 if a.precision == "fp32" else lb.BORIS_FP64
    ens = SoaEnsemble(a.n, prec, w.types, w.light_velocity, with_fields=False)
    ens.fill(w.generate(0, a.n, device="cuda"))
    ens.wrap()
    if a.field == "plane_wave":
        pw = w.plane_wave
        f = lb.boris_field_create_plane_wave(pw["E0"], pw["k_hat"], pw["e_hat"], pw["omega"],
                                             pw["k"], pw["phase0"])
    elif a.field == "uniform":
        f = lb.boris_field_create_uniform(w.uniform_E, w.uniform_B)
    else:
        k = synth.OMEGA0 / synth.C_LIGHT
        f = lb.boris_field_create_mdipole(k * math.sqrt(3e21 / synth.C_LIGHT), synth.OMEGA0, k)
    st = torch.cuda.current_stream()
    for _ in range(a.reps):
        lb.boris_push(ens.handle, f, w.dt, a.steps, st)
    torch.cuda.synchronize()
    lb.boris_field_destroy(f)
    ens.close()


if __name__ == "__main__":
    main()
