#!/usr/bin/env python
"""Per-variant measurements of every §8(a) kernel (one JSON line per variant).

    python scripts/bench_variants.py [--quick] > gpurun_out/variants.jsonl

Streaming variants (per-particle fields, one step per launch) are HBM-bound and
reported as achieved GB/s of algorithmic (layout-implied for AoS) bytes against
MEASURED_PEAKS.json; fused analytic variants are ALU-bound and reported as
particle-updates/s and ps per particle-step.  Device-timed with CUDA events on
the launching stream, after warm-up; inputs larger than L2 for the HBM rows.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
import paper_2104_04579_b200 as lb  # noqa: E402
from paper_2104_04579_b200.ensemble import AosEnsemble, SoaEnsemble  # noqa: E402

PREC = {"fp32": lb.BORIS_FP32, "fp64": lb.BORIS_FP64}


def peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6650.0


def make(w, layout, precision, n):
    cls = SoaEnsemble if layout == "soa" else AosEnsemble
    ens = cls(n, PREC[precision], w.types, w.light_velocity,
              with_fields=w.field_kind == "arrays")
    chunk = 1 << 24
    for c0 in range(0, n, chunk):
        ens.fill(w.generate(c0, min(chunk, n - c0), device="cuda"), first=c0)
    ens.wrap()
    if w.field_kind == "arrays":
        field = ens.field
    elif w.field_kind == "uniform":
        field = lb.boris_field_create_uniform(w.uniform_E, w.uniform_B)
    elif w.field_kind == "plane_wave":
        pw = w.plane_wave
        field = lb.boris_field_create_plane_wave(pw["E0"], pw["k_hat"], pw["e_hat"], pw["omega"],
                                                 pw["k"], pw["phase0"])
    else:
        md = w.plane_wave
        field = lb.boris_field_create_mdipole(md["A0"], md["omega0"], md["k"])
    torch.cuda.synchronize()
    return ens, field


def time_launches(fn, iters, warmup=3):
    st = torch.cuda.current_stream()
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(iters)]
    for a, b in evs:
        a.record(st)
        fn()
        b.record(st)
    torch.cuda.synchronize()
    return statistics.mean(a.elapsed_time(b) for a, b in evs)


def streaming(name, layout, precision, n, diag=False, types=None, iters=20):
    w = synth.config("C2" if not diag else "C5", n=n)
    if types:
        w.types = types
        w.type_mix = "random"
    ens, field = make(w, layout, precision, n)
    fs = 4 if precision == "fp32" else 8
    if layout == "soa":
        bpp = 19 * fs + (2 if types else 0) + (fs if diag else 0)
    else:
        bpp = (36 if fs == 4 else 72) * 2 + 6 * fs
    d = torch.zeros(2, dtype=torch.float64, device="cuda")
    sp = torch.cuda.current_stream().cuda_stream
    if diag:
        fn = lambda: lb.boris_push_diag(ens.handle, field, w.dt, 1, d.data_ptr(), sp)
    else:
        fn = lambda: lb.boris_push(ens.handle, field, w.dt, 1, sp)
    ms = time_launches(fn, iters)
    gbs = bpp * n / (ms * 1e-3) / 1e9
    ens.close()
    return {"variant": name, "layout": layout, "precision": precision, "n": n,
            "field": "per-particle arrays", "steps_per_launch": 1, "diag": diag,
            "n_types": len(w.types), "bytes_per_particle_step": bpp, "ms_per_launch": ms,
            "ps_per_particle_step": ms * 1e9 / n, "achieved_gbs": gbs, "peak_gbs": peak(),
            "frac_of_measured_peak": gbs / peak(), "frac_of_8TBs": gbs / 8000.0}


def fused(name, cfg, layout, precision, n, steps, iters=5, field_kind=None, flags=0):
    w = synth.config(cfg, n=n)
    if field_kind == "mdipole":
        k = synth.OMEGA0 / synth.C_LIGHT
        w.field_kind = "mdipole"
        w.plane_wave = dict(A0=k * math.sqrt(3e21 / synth.C_LIGHT), omega0=synth.OMEGA0, k=k)
    ens, field = make(w, layout, precision, n)
    sp = torch.cuda.current_stream().cuda_stream
    ms = time_launches(lambda: lb.boris_push_ex(ens.handle, field, w.dt, steps, flags, None, sp),
                       iters, warmup=1)
    ens.close()
    lb.boris_field_destroy(field)
    ups = n * steps / (ms * 1e-3)
    return {"variant": name, "layout": layout, "precision": precision, "n": n,
            "field": w.field_kind, "steps_per_launch": steps, "n_types": len(w.types),
            "pusher": {0: "boris", lb.BORIS_PUSH_PUSHER_VAY: "vay",
                       lb.BORIS_PUSH_PUSHER_HIGUERA_CARY: "higuera-cary"}[flags],
            "ms_per_launch": ms, "ps_per_particle_step": 1e12 / ups,
            "particle_updates_per_s": ups}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--fused-only", action="store_true")
    ap.add_argument("--mdipole-only", action="store_true")
    a = ap.parse_args()
    n1 = 10_000_000 if a.quick else 100_000_000
    three = [synth.ELECTRON, synth.POSITRON, synth.PROTON]
    rows = []
    if a.mdipole_only:
        for layout in ("soa", "aos"):
            rows.append(fused(f"mdipole-{layout}-fp32-100", "C4", layout, "fp32", n1 // 4, 100,
                              field_kind="mdipole"))
            rows.append(fused(f"mdipole-{layout}-fp64-100", "C4", layout, "fp64", n1 // 10, 100,
                              field_kind="mdipole"))
        for r in rows:
            print(json.dumps(r), flush=True)
        return
    for n in ([] if a.fused_only else [10_000_000] + ([n1] if n1 != 10_000_000 else [])):
        for layout in ("soa", "aos"):
            for prec in ("fp32", "fp64"):
                rows.append(streaming(f"C2-{layout}-{prec}", layout, prec, n))
        rows.append(streaming("C5-soa-fp32-diag", "soa", "fp32", n, diag=True))
        rows.append(streaming("C2-soa-fp32-3types", "soa", "fp32", n, types=three))
        rows.append(streaming("C2-aos-fp64-3types", "aos", "fp64", n, types=three))
    rows.append(fused("C3-aos-fp64-crossed-100", "C3", "aos", "fp64", 10_000_000, 100))
    rows.append(fused("C4-soa-fp32-planewave-100", "C4", "soa", "fp32", n1, 100))
    rows.append(fused("C4-soa-fp64-planewave-100", "C4", "soa", "fp64", n1 // 4, 100))
    # the same two C4 rows and C3 through the generic (any-orientation) fused kernel
    lb.boris_set_option(lb.BORIS_OPT_FUSED_GENERIC, 1)
    rows.append(fused("C3-aos-fp64-crossed-100-generic", "C3", "aos", "fp64", 10_000_000, 100))
    rows.append(fused("C4-soa-fp32-planewave-100-generic", "C4", "soa", "fp32", n1, 100))
    rows.append(fused("C4-soa-fp64-planewave-100-generic", "C4", "soa", "fp64", n1 // 4, 100))
    lb.boris_set_option(lb.BORIS_OPT_FUSED_GENERIC, 0)
    rows.append(fused("mdipole-soa-fp32-100", "C4", "soa", "fp32", n1 // 4, 100,
                      field_kind="mdipole"))
    rows.append(fused("mdipole-soa-fp64-100", "C4", "soa", "fp64", n1 // 10, 100,
                      field_kind="mdipole"))
    # alternative pushers (generic-orientation fused kernels)
    for pname, fl in (("vay", lb.BORIS_PUSH_PUSHER_VAY),
                      ("hc", lb.BORIS_PUSH_PUSHER_HIGUERA_CARY)):
        rows.append(fused(f"C4-soa-fp32-planewave-100-{pname}", "C4", "soa", "fp32", n1, 100,
                          flags=fl))
        rows.append(fused(f"C3-aos-fp64-crossed-100-{pname}", "C3", "aos", "fp64", 10_000_000,
                          100, flags=fl))
    for r in rows:
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
