#!/usr/bin/env python
"""NEXT row 2: the paper's own benchmark on one B200.

PAPER.md L427-434: 10^7 electrons, initially at rest, uniform in a sphere of
radius 0.6 lambda; the standing m-dipole wave at P = 0.1 PW (eq. 14-15, readings
c9-c13); one "iteration" = 10^3 steps; 10 successive iterations are timed (the
first one discarded as warm-up, L437-449); NSPS = mean iteration time /
(10^7 x 10^3).  Cells: {AoS, SoA} x {fp32, fp64} x {precalculated, analytic}
(Table 2).

* precalculated: the m-dipole evaluated at the initial positions at t = T/8
  (boris_field_evaluate; the paper does not say when, reading in DESIGN.md),
  stored per particle and re-read every step (BORIS_PUSH_STREAM_EACH_STEP: one
  streaming launch per step, like the paper's one submit per step, L286-299);
  the extra column "precalc fused" is the same push with BORIS_PUSH_AUTO
  (bitwise-identical results, fields read once per iteration).
* analytic: the m-dipole evaluated inline, 10^3 steps fused in registers.

dt is not given by the paper (reading c7): T/10^4 here.
Prints one JSON line per cell and a markdown table beside the paper's Xeon
numbers (context, not a target).
"""
import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
import paper_2104_04579_b200 as lb  # noqa: E402
from paper_2104_04579_b200.ensemble import AosEnsemble, SoaEnsemble  # noqa: E402

# Table 2 (L460-471), 2x Xeon Platinum 8260L, best of OpenMP / DPC++ / DPC++ NUMA, NSPS.
PAPER_XEON = {
    ("aos", "fp32", "precalc"): 0.53, ("aos", "fp64", "precalc"): 0.98,
    ("aos", "fp32", "analytic"): 0.54, ("aos", "fp64", "analytic"): 0.84,
    ("soa", "fp32", "precalc"): 0.50, ("soa", "fp64", "precalc"): 1.06,
    ("soa", "fp32", "analytic"): 0.43, ("soa", "fp64", "analytic"): 0.76,
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=10_000_000)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--only", default=None, help="run one scenario (precalc, precalc fused, "
                                                  "analytic)")
    a = ap.parse_args()
    k = synth.OMEGA0 / synth.C_LIGHT
    A0 = k * math.sqrt(3.0 * 1e21 / synth.C_LIGHT)   # reading c12, P = 0.1 PW = 1e21 erg/s
    w = synth.Workload("paper", a.n, 7, [synth.ELECTRON], synth.T0 / 1e4, a.steps,
                       field_kind="mdipole")
    md = lb.boris_field_create_mdipole(A0, synth.OMEGA0, k)
    st = torch.cuda.current_stream()
    rows = []
    for layout in ("aos", "soa"):
        for prec in ("fp32", "fp64"):
            p = lb.BORIS_FP32 if prec == "fp32" else lb.BORIS_FP64
            cls = SoaEnsemble if layout == "soa" else AosEnsemble
            ens = cls(a.n, p, w.types, w.light_velocity, with_fields=True)
            d0 = w.generate(0, a.n, device="cuda")
            for scenario, flags in (("precalc", lb.BORIS_PUSH_STREAM_EACH_STEP),
                                    ("precalc fused", lb.BORIS_PUSH_AUTO),
                                    ("analytic", None)):
                if a.only is not None and scenario != a.only:
                    continue
                ens.fill(d0)
                ens.wrap()
                if flags is not None:
                    lb.boris_field_evaluate(md, ens.handle, synth.T0 / 8, ens.field, st)
                times = []
                for it in range(a.iters + 1):
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record(st)
                    if flags is None:
                        lb.boris_push(ens.handle, md, w.dt, a.steps, st)
                    else:
                        lb.boris_push_ex(ens.handle, ens.field, w.dt, a.steps, flags, None, st)
                    e1.record(st)
                    torch.cuda.synchronize()
                    if it > 0:     # first iteration discarded (L437-449)
                        times.append(e0.elapsed_time(e1))
                ms = sum(times) / len(times)
                nsps = ms * 1e6 / (a.n * a.steps)
                key = (layout, prec, "precalc" if scenario.startswith("precalc") else "analytic")
                row = {"layout": layout, "precision": prec, "scenario": scenario,
                       "particles": a.n, "steps_per_iteration": a.steps, "iterations": a.iters,
                       "ms_per_iteration": ms, "nsps": nsps,
                       "paper_xeon_nsps": PAPER_XEON[key],
                       "speedup_vs_paper_xeon": PAPER_XEON[key] / nsps}
                rows.append(row)
                print(json.dumps(row), flush=True)
            ens.close()
    lb.boris_field_destroy(md)
    print("\n| layout | FP | scenario | B200 NSPS | paper 2x Xeon 8260L NSPS (L460-471) | ratio |")
    print("|---|---|---|---|---|---|")
    for r in rows:
        print(f"| {r['layout']} | {r['precision']} | {r['scenario']} | {r['nsps']:.5f} | "
              f"{r['paper_xeon_nsps']:.2f} | {r['speedup_vs_paper_xeon']:.0f}x |")


if __name__ == "__main__":
    main()
