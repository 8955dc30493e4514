#!/usr/bin/env python
"""Table-2 analytic m-dipole cells, SoA only (variant sweeps): 10^7 electrons in the
0.6-lambda sphere, P = 0.1 PW, 10^3 fused steps per iteration, mean of `--iters`
after one discarded.  One JSON line per precision, tagged with
the loaded library (LIBBORIS_PATH selects a tuning build).

    LIBBORIS_PATH=... python scripts/bench_md.py [--tag NAME]
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
from paper_2104_04579_b200.ensemble import SoaEnsemble  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=10_000_000)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--tag", default=os.path.basename(os.environ.get("LIBBORIS_PATH", "libboris.so")))
    ap.add_argument("--precisions", default="fp32,fp64")
    a = ap.parse_args()
    k = synth.OMEGA0 / synth.C_LIGHT
    A0 = k * math.sqrt(3.0 * 1e21 / synth.C_LIGHT)
    w = synth.Workload("paper", a.n, 7, [synth.ELECTRON], synth.T0 / 1e4, a.steps,
                       field_kind="mdipole")
    md = lb.boris_field_create_mdipole(A0, synth.OMEGA0, k)
    st = torch.cuda.current_stream()
    for prec in a.precisions.split(","):
        p = lb.BORIS_FP32 if prec == "fp32" else lb.BORIS_FP64
        ens = SoaEnsemble(a.n, p, w.types, w.light_velocity, with_fields=False)
        ens.fill(w.generate(0, a.n, device="cuda"))
        ens.wrap()
        times = []
        for it in range(a.iters + 1):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(st)
            lb.boris_push(ens.handle, md, w.dt, a.steps, st)
            e1.record(st)
            torch.cuda.synchronize()
            if it > 0:
                times.append(e0.elapsed_time(e1))
        ms = sum(times) / len(times)
        print(json.dumps({"tag": a.tag, "precision": prec, "n": a.n, "steps": a.steps,
                          "ms": ms, "ps_per_particle_step": ms * 1e9 / (a.n * a.steps),
                          "times_ms": times}), flush=True)
        ens.close()
    lb.boris_field_destroy(md)


if __name__ == "__main__":
    main()
