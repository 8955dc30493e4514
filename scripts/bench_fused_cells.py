#!/usr/bin/env python
"""C3 / C4 / Table-2 m-dipole fused cells (bench.py's recipes) for variant sweeps: one
JSON line per cell, tagged with the loaded library (LIBBORIS_PATH selects a tuning build).

    LIBBORIS_PATH=... python scripts/bench_fused_cells.py [--cells C3,C4,md64,md32]
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


def cell(name, cfg, layout, prec, n, steps, mdipole, iters, tag):
    w = synth.config(cfg, n=n)
    if mdipole:
        k = synth.OMEGA0 / synth.C_LIGHT
        w.field_kind = "mdipole"
        w.plane_wave = dict(A0=k * math.sqrt(3e21 / synth.C_LIGHT), omega0=synth.OMEGA0, k=k)
        w.dt = synth.T0 / 1e4
    p = lb.BORIS_FP32 if prec == "fp32" else lb.BORIS_FP64
    cls = SoaEnsemble if layout == "soa" else AosEnsemble
    ens = cls(n, p, w.types, w.light_velocity, with_fields=False)
    ens.fill(w.generate(0, n, device="cuda"))
    ens.wrap()
    if w.field_kind == "uniform":
        field = lb.boris_field_create_uniform(w.uniform_E, w.uniform_B)
    elif w.field_kind == "plane_wave":
        pw = w.plane_wave
        field = lb.boris_field_create_plane_wave(pw["E0"], pw["k_hat"], pw["e_hat"], pw["omega"],
                                                 pw["k"], pw["phase0"])
    else:
        md = w.plane_wave
        field = lb.boris_field_create_mdipole(md["A0"], md["omega0"], md["k"])
    st = torch.cuda.current_stream()
    times = []
    for it in range(iters + 1):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(st)
        lb.boris_push(ens.handle, field, w.dt, steps, st)
        b.record(st)
        torch.cuda.synchronize()
        if it:
            times.append(a.elapsed_time(b))
    ms = sum(times) / len(times)
    print(json.dumps({"tag": tag, "cell": name, "n": n, "steps": steps, "ms": ms,
                      "ps_per_particle_step": ms * 1e9 / (n * steps)}), flush=True)
    lb.boris_field_destroy(field)
    ens.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cells", default="C3,C4,md64,md32")
    ap.add_argument("--tag", default=os.path.basename(os.environ.get("LIBBORIS_PATH",
                                                                     "libboris.so")))
    a = ap.parse_args()
    cells = {
        "C3": ("C3", "aos", "fp64", 10_000_000, 100, False, 5),
        "C4": ("C4", "soa", "fp32", 100_000_000, 100, False, 5),
        "md64": ("C4", "soa", "fp64", 10_000_000, 1000, True, 2),
        "md32": ("C4", "soa", "fp32", 10_000_000, 1000, True, 2),
    }
    for c in a.cells.split(","):
        cell(c, *cells[c], tag=a.tag)


if __name__ == "__main__":
    main()
