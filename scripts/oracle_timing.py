#!/usr/bin/env python
"""Oracle timing on the host cores (SURVEY §8(d) "Oracle timing in the same run"):
the scalar double C oracle, as it stands, on C2 (per-particle fields) and C4
(plane wave) subsets, single-threaded and with all cores (the paper's loop shape:
steps outside, OpenMP over particles, L256-269).  A baseline only, never a target.

    python scripts/oracle_timing.py [--n 1000000] [--seconds 8]

Prints the host description (nproc, lscpu model/sockets/cores/threads) and one
JSON line per (workload, threads) with ns/particle/step.
"""
import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
from parity_util import oracle_field, stack3  # noqa: E402


def host():
    info = {"nproc": os.cpu_count()}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
        for line in out.splitlines():
            k, _, v = line.partition(":")
            if k.strip() in ("Model name", "Socket(s)", "Core(s) per socket",
                             "Thread(s) per core", "NUMA node(s)"):
                info[k.strip()] = v.strip()
    except OSError:
        pass
    return info


def run(name, n, threads, seconds):
    w = synth.config(name, n=n)
    d = w.generate(0, n)
    pos, mom = stack3(d, "x", "y", "z"), stack3(d, "px", "py", "pz")
    typ = d["type"].numpy().astype(np.int16)
    tq, tm = [t[0] for t in w.types], [t[1] for t in w.types]
    kind, params = oracle_field(w, "fp64")
    kw = dict(params=params, dt=w.dt, n_threads=threads)
    if kind == oracle.FIELD_ARRAYS:
        kw.update(E=stack3(d, "Ex", "Ey", "Ez"), B=stack3(d, "Bx", "By", "Bz"))
    oracle.push(pos, mom, typ, tq, tm, w.light_velocity, kind, n_steps=2, **kw)  # warm-up
    t0 = time.perf_counter()
    oracle.push(pos, mom, typ, tq, tm, w.light_velocity, kind, n_steps=4, **kw)
    per = (time.perf_counter() - t0) / 4
    steps = max(1, min(5000, int(seconds / max(per, 1e-9))))
    t0 = time.perf_counter()
    oracle.push(pos, mom, typ, tq, tm, w.light_velocity, kind, n_steps=steps, **kw)
    el = time.perf_counter() - t0
    return {"exp": "oracle_timing", "workload": name, "field": w.field_kind, "n": n,
            "threads": threads, "steps": steps, "seconds": el,
            "ns_per_particle_step": el * 1e9 / (n * steps),
            "particle_updates_per_s": n * steps / el}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--seconds", type=float, default=8.0)
    a = ap.parse_args()
    print(json.dumps({"exp": "host", **host()}), flush=True)
    logical = os.cpu_count() or 1
    for name in ("C2", "C4"):
        for threads in sorted({1, max(1, logical // 2), logical}):
            print(json.dumps(run(name, a.n, threads, a.seconds)), flush=True)


if __name__ == "__main__":
    torch.set_num_threads(1)
    main()
