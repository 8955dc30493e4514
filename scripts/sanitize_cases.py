#!/usr/bin/env python
"""Every libboris kernel variant on small ragged inputs, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck).  Exits 0 when every call
succeeds; the sanitizer's own exit code reports hazards.

    compute-sanitizer --tool racecheck --error-exitcode 9 python scripts/sanitize_cases.py
"""
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2104_04579_b200 as lb  # noqa: E402
from paper_2104_04579_b200.ensemble import AosEnsemble, SoaEnsemble  # noqa: E402

THREE = [synth.ELECTRON, synth.POSITRON, synth.PROTON]


def analytic(kind):
    k = synth.OMEGA0 / synth.C_LIGHT
    if kind == "uniform":
        return lb.boris_field_create_uniform([0, 0.5 * synth.B0, 0], [0, 0, synth.B0])
    if kind == "plane_wave":
        return lb.boris_field_create_plane_wave(10 * synth.E_UNIT, [1, 0, 0], [0, 1, 0],
                                                synth.OMEGA0, k, 0.0)
    return lb.boris_field_create_mdipole(k * math.sqrt(3e21 / synth.C_LIGHT), synth.OMEGA0, k)


def main():
    d_diag = torch.zeros(2, dtype=torch.float64, device="cuda")
    dp = d_diag.data_ptr()
    for n in (1, 13, 4096 + 13):
        for prec in (lb.BORIS_FP32, lb.BORIS_FP64):
            for types in ([synth.ELECTRON], THREE):
                w = synth.config("C5", n=n)
                w.types = types
                w.type_mix = "random"
                d = w.generate()
                for cls in (SoaEnsemble, AosEnsemble):
                    e = cls(n, prec, types, w.light_velocity)
                    e.fill(d)
                    e.wrap()
                    lb.boris_push(e.handle, e.field, w.dt, 1)                  # streaming
                    lb.boris_push_diag(e.handle, e.field, w.dt, 1, dp)         # streaming + KE
                    lb.boris_push_ex(e.handle, e.field, w.dt, 3, lb.BORIS_PUSH_AUTO, dp)
                    lb.boris_kinetic_energy(e.handle, dp)
                    for kind in ("uniform", "plane_wave", "mdipole"):
                        f = analytic(kind)
                        lb.boris_push_diag(e.handle, f, w.dt, 9, dp)           # fused analytic
                        lb.boris_field_evaluate(f, e.handle, 0.1 * synth.T0, e.field)
                        lb.boris_field_destroy(f)
                    torch.cuda.synchronize()
                    e.close()
                # unaligned SoA (scalar path)
                if n > 1:
                    big = SoaEnsemble(n, prec, types, w.light_velocity)
                    big.fill(d)
                    keys = ("x", "y", "z", "px", "py", "pz")
                    h = lb.boris_ensemble_wrap_soa(
                        0, lb.BORIS_MEMORY_DEVICE, prec, n - 1, *(big.t[k][1:].data_ptr() for k in keys),
                        big.t["weight"][1:].data_ptr(), big.t["gamma"][1:].data_ptr(),
                        big.t["type"][1:].data_ptr() if big.t["type"] is not None else None,
                        types, w.light_velocity)
                    f = lb.boris_field_create_arrays_soa(
                        h, *(big.t[k][1:].data_ptr() for k in ("Ex", "Ey", "Ez", "Bx", "By", "Bz")))
                    lb.boris_push_diag(h, f, w.dt, 1, dp)
                    torch.cuda.synchronize()
                    lb.boris_field_destroy(f)
                    lb.boris_ensemble_destroy(h)
        # owned ensemble upload / download
        h = lb.boris_ensemble_create(0, lb.BORIS_LAYOUT_AOS, lb.BORIS_FP64, n, THREE, synth.C_LIGHT)
        pos = np.random.default_rng(1).normal(size=(n, 3))
        lb.boris_ensemble_upload(h, 0, n, pos, pos * 1e-17, np.ones(n), np.zeros(n, np.int16))
        lb.boris_ensemble_download(h, 0, n)
        lb.boris_ensemble_destroy(h)
    # grid gather push, sort by cell, deposition, alternative pushers (NEXT rows 3-4)
    for prec in (lb.BORIS_FP32, lb.BORIS_FP64):
        dt = torch.float32 if prec == lb.BORIS_FP32 else torch.float64
        g = 5
        L = 1.5 * synth.LAMBDA0
        comps = [torch.randn((g, g + 1, g + 2), device="cuda", dtype=torch.float64).to(dt)
                 * synth.E_UNIT for _ in range(6)]
        grid = lb.boris_field_create_grid(0, prec, g + 2, g + 1, g, [-L / 2] * 3,
                                          [L / (g + 2), L / (g + 1), L / g],
                                          *(c.data_ptr() for c in comps))
        J = [torch.zeros((g, g + 1, g + 2), device="cuda", dtype=dt) for _ in range(3)]
        for n, types in ((13, THREE), (3 * 2048 + 77, THREE), (3 * 2048 + 77, [synth.ELECTRON])):
            w = synth.config("C2", n=n)
            w.types = types
            w.type_mix = "random"
            for cls in (SoaEnsemble, AosEnsemble):
                e = cls(n, prec, types, w.light_velocity)
                e.fill(w.generate())
                e.wrap()
                lb.boris_ensemble_sort_by_cell(e.handle, grid)
                lb.boris_push_diag(e.handle, grid, w.dt, 3, dp)
                lb.boris_push_diag(e.handle, grid, w.dt, 1, dp)   # streaming grid step
                lb.boris_deposit_current(e.handle, grid, w.dt, *(j.data_ptr() for j in J))
                lb.boris_push_deposit(e.handle, grid, w.dt, *(j.data_ptr() for j in J), dp)
                lb.boris_push_deposit(e.handle, grid, w.dt, *(j.data_ptr() for j in J))
                lb.boris_field_evaluate(grid, e.handle, 0.0, e.field)
                for flags in (lb.BORIS_PUSH_PUSHER_VAY, lb.BORIS_PUSH_PUSHER_HIGUERA_CARY):
                    lb.boris_push_ex(e.handle, e.field, w.dt, 2, flags, dp)
                    lb.boris_push_ex(e.handle, grid, w.dt, 2, flags, dp)
                    f = analytic("plane_wave")
                    lb.boris_push_ex(e.handle, f, w.dt, 2, flags, dp)
                    lb.boris_field_destroy(f)
                for generic in (0, 1):   # axis-aligned specialisation and generic
                    lb.boris_set_option(lb.BORIS_OPT_FUSED_GENERIC, generic)
                    for kind in ("uniform", "plane_wave"):
                        f = analytic(kind)
                        lb.boris_push_diag(e.handle, f, w.dt, 11, dp)
                        lb.boris_field_destroy(f)
                lb.boris_set_option(lb.BORIS_OPT_FUSED_GENERIC, 0)
                torch.cuda.synchronize()
                e.close()
        # wrapped SoA one element off alignment (scalar / warp-run paths), no weight
        n = 2 * 2048 + 45
        big = SoaEnsemble(n + 1, prec, THREE, synth.C_LIGHT)
        wv = synth.config("C2", n=n + 1)
        wv.types = THREE
        wv.type_mix = "random"
        big.fill(wv.generate())
        keys = ("x", "y", "z", "px", "py", "pz")
        h = lb.boris_ensemble_wrap_soa(0, lb.BORIS_MEMORY_DEVICE, prec, n,
                                       *(big.t[k][1:].data_ptr() for k in keys), None,
                                       big.t["gamma"][1:].data_ptr(), big.t["type"][1:].data_ptr(),
                                       THREE, synth.C_LIGHT)
        lb.boris_ensemble_sort_by_cell(h, grid)
        lb.boris_deposit_current(h, grid, wv.dt, *(j.data_ptr() for j in J))
        lb.boris_push_deposit(h, grid, wv.dt, *(j.data_ptr() for j in J), dp)
        torch.cuda.synchronize()
        lb.boris_ensemble_destroy(h)
        big.close()
        lb.boris_field_destroy(grid)
    # the full 256-entry type table (shared-memory copy in every multi-type kernel)
    many = [(synth.E_CHARGE * (1 - 2 * (i % 2)), synth.M_ELECTRON * (1 + i)) for i in range(256)]
    w = synth.config("C2", n=4096 + 7)
    w.types = many
    w.type_mix = "random"
    for cls in (SoaEnsemble, AosEnsemble):
        e = cls(w.n, lb.BORIS_FP32, many, w.light_velocity)
        e.fill(w.generate())
        e.wrap()
        lb.boris_push_diag(e.handle, e.field, w.dt, 1, dp)
        lb.boris_push_diag(e.handle, e.field, w.dt, 4, dp)
        torch.cuda.synchronize()
        e.close()
    # host-resident pipeline, several chunks
    lb.boris_set_option(lb.BORIS_OPT_HOST_CHUNK, 2048)
    w = synth.config("C5", n=5000)
    for cls in (SoaEnsemble, AosEnsemble):
        e = cls(w.n, lb.BORIS_FP32, w.types, w.light_velocity, host=True)
        e.fill(w.generate())
        e.wrap()
        lb.boris_push_diag(e.handle, e.field, w.dt, 2, dp)
        torch.cuda.synchronize()
        e.close()
    print("sanitize cases: ok")


if __name__ == "__main__":
    main()
