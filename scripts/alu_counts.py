#!/usr/bin/env python
"""Executed-instruction counts of the register-fused kernels, for their ALU rooflines.

    ncu --metrics smsp__inst_executed.sum,smsp__inst_executed_pipe_xu.sum,\
smsp__inst_executed_pipe_fp64.sum,gpu__time_duration.sum --csv \
        --log-file gpurun_out/alu.csv python scripts/alu_counts.py run
    python scripts/alu_counts.py parse gpurun_out/alu.csv > profiles/alu_counts.json

`run` launches each fused configuration bench.py measures (same kernels, same field
parameters, smaller n) once, in a fixed order; `parse` divides the ncu counts by the
warp-steps of each launch (n/32 x steps) and writes the per-kernel figures bench.py's
alu_bound_ps() turns into a lower bound on ps per particle-step.
"""
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

# (key, cfg, layout, precision, n, steps, mdipole) -- the order of the launches
CASES = [
    ("C3_aos_fp64_uniform_yz", "C3", "aos", "fp64", 1_048_576, 100, False),
    ("C4_soa_fp32_planewave_yz", "C4", "soa", "fp32", 4_194_304, 100, False),
    ("mdipole_soa_fp32", "C4", "soa", "fp32", 1_048_576, 1000, True),
    ("mdipole_aos_fp32", "C4", "aos", "fp32", 1_048_576, 1000, True),
    ("mdipole_soa_fp64", "C4", "soa", "fp64", 1_048_576, 1000, True),
    ("mdipole_aos_fp64", "C4", "aos", "fp64", 1_048_576, 1000, True),
]


def run():
    import torch
    import synth
    import paper_2104_04579_b200 as lb
    from paper_2104_04579_b200.ensemble import AosEnsemble, SoaEnsemble
    sp = torch.cuda.current_stream().cuda_stream
    for key, cfg, layout, prec, n, steps, md in CASES:
        w = synth.config(cfg, n=n)
        if md:
            k = synth.OMEGA0 / synth.C_LIGHT
            w.field_kind = "mdipole"
            w.plane_wave = dict(A0=k * math.sqrt(3e21 / synth.C_LIGHT), omega0=synth.OMEGA0, k=k)
            w.dt = synth.T0 / 1e4
        cls = SoaEnsemble if layout == "soa" else AosEnsemble
        ens = cls(n, lb.BORIS_FP32 if prec == "fp32" else lb.BORIS_FP64, w.types,
                  w.light_velocity, with_fields=False)
        ens.fill(w.generate(0, n, device="cuda"))
        ens.wrap()
        if w.field_kind == "uniform":
            f = lb.boris_field_create_uniform(w.uniform_E, w.uniform_B)
        elif w.field_kind == "plane_wave":
            pw = w.plane_wave
            f = lb.boris_field_create_plane_wave(pw["E0"], pw["k_hat"], pw["e_hat"], pw["omega"],
                                                 pw["k"], pw["phase0"])
        else:
            mdp = w.plane_wave
            f = lb.boris_field_create_mdipole(mdp["A0"], mdp["omega0"], mdp["k"])
        lb.boris_push(ens.handle, f, w.dt, steps, sp)
        torch.cuda.synchronize()
        print(key, flush=True)
        lb.boris_field_destroy(f)
        ens.close()


def parse(path):
    import csv
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    per = {}
    for r in rows[1:]:
        if "k_fused" not in r[ix["Kernel Name"]]:
            continue
        per.setdefault(r[ix["ID"]], {"name": r[ix["Kernel Name"]]})[r[ix["Metric Name"]]] = \
            float(r[ix["Metric Value"]].replace(",", ""))
    launches = [per[k] for k in sorted(per, key=int)]
    launches = [l for l in launches if "k_diag" not in l["name"]]
    out = {"source": os.path.basename(path), "how": "ncu executed warp-instructions of one "
           "launch / (n/32 x steps); scripts/alu_counts.py", "kernels": {}}
    # a push of > 1024 m-dipole steps is split into launches: sum them per case
    i = 0
    for key, cfg, layout, prec, n, steps, md in CASES:
        nl = -(-steps // 1024) if md else 1
        ls = launches[i:i + nl]
        i += nl
        ws = n / 32 * steps
        tot = lambda m: sum(l[m] for l in ls)
        out["kernels"][key] = {
            "kernel": ls[0]["name"][:120], "n": n, "steps": steps,
            "inst_per_warp_step": tot("smsp__inst_executed.sum") / ws,
            "xu_per_warp_step": tot("smsp__inst_executed_pipe_xu.sum") / ws,
            "fp64_per_warp_step": tot("smsp__inst_executed_pipe_fp64.sum") / ws,
            "ncu_ps_per_particle_step": tot("gpu__time_duration.sum") * 1e3 / (n * steps)
            if "gpu__time_duration.sum" in ls[0] else None}
    json.dump(out, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run()
    else:
        parse(sys.argv[2])
