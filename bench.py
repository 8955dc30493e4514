#!/usr/bin/env python
"""Benchmark of the B200 Boris pusher (libboris) -- prints ONE JSON line.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl libboris|reference]
                    [--workload C5|C2|C4] [--particles N_total]

Default workload: BASELINE.json configs[4] ("C5"): 8e8 particles in total,
sharded over the ranks (strong scaling), per-particle E/B fields, fp32 SoA, one
Boris step per launch, with the per-step kinetic-energy diagnostic allreduced
over ranks (NCCL).  A step = one pass of the whole hot path (SURVEY §8(a) rows
a1-a13) over the ensemble.  Inputs (8e8 x 80 B) are far larger than L2 (126 MB).

Multi-GPU: launched by torchrun (RANK / WORLD_SIZE / LOCAL_RANK), one process
per GPU; device-timed with CUDA events, max over ranks.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = ("ns/particle/step (particle updates/s) and achieved HBM GB/s vs 8 TB/s, "
          "1/2/4/8 GPU")
# Algorithmic bytes per particle-step of the timed kernel:
# fp32 SoA: read r,p (24) + E,B (24) + weight (4, KE diag); write r,p (24) + gamma (4).
BYTES_PER_PARTICLE_STEP = {"C5": 80, "C2": 76}
FALLBACK_HBM_GBS = 6650.0


def measured_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled DURING the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm, smax, reasons = [], [], set()
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for name, val in zip(self.NAMES, parts[2:6]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_baseline(workload, target_s=15.0, sample=1 << 21, threads=None):
    """The oracle (as it stands) on the host cores, on a bounded sample of the workload."""
    import numpy as np
    import torch
    import oracle
    threads = threads or os.cpu_count() or 1
    d = workload.generate(0, sample)
    d = {k: (v.to(torch.float32).to(torch.float64) if v.dtype == torch.float64 else v)
         for k, v in d.items()}
    st = lambda a, b, c: torch.stack([d[a], d[b], d[c]], 1).numpy()
    pos, mom = st("x", "y", "z"), st("px", "py", "pz")
    E, B = st("Ex", "Ey", "Ez"), st("Bx", "By", "Bz")
    args = (pos, mom, d["type"].numpy(), [workload.types[0][0]], [workload.types[0][1]],
            workload.light_velocity, oracle.FIELD_ARRAYS)
    oracle.push(*args, E=E, B=B, dt=workload.dt, n_steps=1, n_threads=threads)  # warm-up
    t0 = time.perf_counter()
    oracle.push(*args, E=E, B=B, dt=workload.dt, n_steps=8, n_threads=threads)
    t1 = (time.perf_counter() - t0) / 8          # steady per-step time (calibration)
    steps = int(max(1, min(4000, target_s / max(t1, 1e-6))))
    t0 = time.perf_counter()
    oracle.push(*args, E=E, B=B, dt=workload.dt, n_steps=steps, n_threads=threads)
    el = time.perf_counter() - t0
    return {"value": sample * steps / el, "unit": "particle-updates/s", "cores": threads,
            "kind": "oracle",
            "sample": f"{sample} particles x {steps} steps of {workload.name} (fp64 scalar C "
                      f"oracle, per-particle fields, OpenMP {threads} threads, {el:.1f} s)"}


def arm_config(w, n_local, world, bpp):
    """The `config` object of the JSON line (the same for both arms)."""
    return {"workload": f"{w.name}: BASELINE configs[4]" if w.name == "C5" else w.name,
            "particles_total": w.n, "particles_per_gpu": n_local,
            "layout": "SoA", "field": "per-particle E/B arrays",
            "steps_per_launch": 1, "diagnostic": "per-step KE + count allreduce",
            "parallelism": f"shard{world}", "l2": "inputs larger than L2 "
            f"({bpp * n_local / 1e9:.1f} GB per GPU per step vs 126 MB)"}


def run_reference(args):
    """--impl reference: the oracle timed as the reference arm (rank 0 only)."""
    rank = int(os.environ.get("RANK", 0))
    if rank != 0:
        return 0
    import numpy as np
    import torch
    import synth
    import oracle
    w = synth.config(args.workload, n=args.particles)
    world = int(os.environ.get("WORLD_SIZE", args.gpus))
    threads = os.cpu_count() or 1
    sample = args.ref_sample
    d = w.generate(0, sample)
    d = {k: (v.to(torch.float32).to(torch.float64) if v.dtype == torch.float64 else v)
         for k, v in d.items()}
    st = lambda a, b, c: torch.stack([d[a], d[b], d[c]], 1).numpy()
    pos, mom = st("x", "y", "z"), st("px", "py", "pz")
    E, B = st("Ex", "Ey", "Ez"), st("Bx", "By", "Bz")
    typ = d["type"].numpy()
    tq, tm = [w.types[0][0]], [w.types[0][1]]
    for _ in range(args.warmup):
        pos, mom, g = oracle.push(pos, mom, typ, tq, tm, w.light_velocity, oracle.FIELD_ARRAYS,
                                  E=E, B=B, dt=w.dt, n_steps=1, n_threads=threads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        pos, mom, g = oracle.push(pos, mom, typ, tq, tm, w.light_velocity, oracle.FIELD_ARRAYS,
                                  E=E, B=B, dt=w.dt, n_steps=1, n_threads=threads)
        ke = oracle.kinetic_energy(mom, g, d["weight"].numpy(), typ, tm, w.light_velocity)
    el = time.perf_counter() - t0
    value = sample * args.steps / el
    unit = "particle-updates/s"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": unit,
        "n_gpus": int(os.environ.get("WORLD_SIZE", args.gpus)), "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "ns_per_particle_step": 1e9 / value,
        "config": arm_config(w, w.n // world - (w.n // world) % 8, world,
                             BYTES_PER_PARTICLE_STEP[w.name]),
        "cpu_baseline": {"value": value, "unit": unit, "cores": threads, "kind": "oracle",
                         "sample": f"{sample} particles x {args.steps} steps of {w.name} (fp64 "
                                   "scalar C oracle, canonical double layout, per-particle "
                                   "fields, OpenMP over the host cores; throughput scales "
                                   "linearly in the particle count)"},
        "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="libboris", choices=["libboris", "reference"])
    ap.add_argument("--workload", default="C5", choices=["C5", "C2"])
    ap.add_argument("--particles", type=int, default=None, help="global particle count")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-sample", type=int, default=1 << 20)
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import synth
    import paper_2104_04579_b200 as lb
    from paper_2104_04579_b200 import dist as bdist
    from paper_2104_04579_b200.ensemble import SoaEnsemble

    # one process per GPU; BORIS_DIST_BACKEND=gloo + BORIS_SHARE_GPU=1 lets a 1-GPU box run
    # the N>1 code path (all ranks on cuda:0) for testing -- never for a reported number.
    local = int(os.environ.get("LOCAL_RANK", 0))
    if os.environ.get("BORIS_SHARE_GPU") == "1":
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    rank, world = bdist.init(os.environ.get("BORIS_DIST_BACKEND", "nccl"))
    dev = torch.device("cuda", local)
    lb.load_library()

    w = synth.config(args.workload, n=args.particles)
    lo, hi = bdist.shard_range(w.n, rank, world)
    n_local = hi - lo
    bpp = BYTES_PER_PARTICLE_STEP[w.name]

    # ---- device-resident ensemble, generated on the GPU by global index ----
    ens = SoaEnsemble(n_local, lb.BORIS_FP32, w.types, w.light_velocity, device=local)
    chunk = 1 << 24
    for c0 in range(lo, hi, chunk):
        cnt = min(chunk, hi - c0)
        ens.fill(w.generate(c0, cnt, device=dev), first=c0 - lo)
    ens.wrap()
    torch.cuda.synchronize()

    stream = torch.cuda.current_stream()
    sptr = stream.cuda_stream
    diag = [torch.zeros(2, dtype=torch.float64, device=dev) for _ in range(2)]
    works = [None, None]

    def step(k, ev_a=None, ev_b=None):
        buf = k % 2
        if works[buf] is not None:
            works[buf].wait()
        if ev_a is not None:
            ev_a.record(stream)
        lb.boris_push_diag(ens.handle, ens.field, w.dt, 1, diag[buf].data_ptr(), sptr)
        if ev_b is not None:
            ev_b.record(stream)
        if world > 1:
            works[buf] = torch.distributed.all_reduce(diag[buf], async_op=True)

    for k in range(args.warmup):
        step(k)
    for wk in works:
        if wk is not None:
            wk.wait()
    works = [None, None]
    torch.cuda.synchronize()
    bdist.barrier(dev)

    clocks = ClockSampler(local).start()
    time.sleep(0.2)
    ev_a = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ev_b = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    bdist.barrier(dev)
    start.record(stream)
    for k in range(args.steps):
        step(k, ev_a[k], ev_b[k])
    for wk in works:
        if wk is not None:
            wk.wait()
    end.record(stream)
    torch.cuda.synchronize()
    bdist.barrier(dev)
    clk = clocks.stop()
    elapsed_ms = bdist.max_over_ranks(start.elapsed_time(end), dev)
    push_ms = statistics.mean(a.elapsed_time(b) for a, b in zip(ev_a, ev_b))
    push_ms_max = bdist.max_over_ranks(push_ms, dev)
    final_diag = diag[(args.steps - 1) % 2].tolist()

    ms_per_step = elapsed_ms / args.steps
    value = w.n * args.steps / (elapsed_ms * 1e-3)            # whole-job particle-updates/s
    peak, peak_kind = measured_peak()
    achieved = bpp * n_local / (push_ms * 1e-3) / 1e9         # GB/s of the push kernel
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        try:
            tj = json.load(open(tpath))
            ent = tj.get(f"{w.name}:n_local={n_local}")
            if ent:
                traffic = ent["dram_bytes_per_launch"]
        except Exception:
            traffic = None

    # ---- end to end: host-resident (pinned) ensemble through the public C ABI ----
    e2e = None
    if not args.no_e2e:
        hens = SoaEnsemble(n_local, lb.BORIS_FP32, w.types, w.light_velocity, host=True)
        for k2, v in ens.t.items():
            if v is not None:
                hens.t[k2].copy_(v)
        hens.wrap()
        hdiag = torch.zeros(2, dtype=torch.float64, device=dev)
        out = torch.zeros(2, dtype=torch.float64, pin_memory=True)
        torch.cuda.synchronize()
        for _ in range(1):  # warm-up (allocates the staging pipeline)
            lb.boris_push_diag(hens.handle, hens.field, w.dt, 1, hdiag.data_ptr(), sptr)
            out.copy_(hdiag, non_blocking=True)
        torch.cuda.synchronize()
        bdist.barrier(dev)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.e2e_steps):
            lb.boris_push_diag(hens.handle, hens.field, w.dt, 1, hdiag.data_ptr(), sptr)
            if world > 1:
                torch.distributed.all_reduce(hdiag)
            out.copy_(hdiag, non_blocking=True)   # D2H read of the step's result
            stream.synchronize()
        e1.record(stream)
        torch.cuda.synchronize()
        e2e_ms = bdist.max_over_ranks(e0.elapsed_time(e1), dev)
        e2e = {"value": w.n * args.e2e_steps / (e2e_ms * 1e-3), "unit": "particle-updates/s",
               "h2d_bytes_per_step": n_local * 52, "d2h_bytes_per_step": n_local * 28 + 16,
               "ms_per_step": e2e_ms / args.e2e_steps,
               "path": "boris_push_diag on a pinned host-resident SoA ensemble: chunked "
                       "H2D(r,p,E,B,w) -> push+KE -> D2H(r,p,gamma) pipeline, + KE readback"}
        hens.close()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(w)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "particle-updates/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "ns_per_particle_step": 1e9 / value,
            "hbm_gbs_per_gpu": achieved,
            "config": arm_config(w, n_local, world, bpp),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "peak_kind": peak_kind, "frac_of_nominal_8tbs": achieved / 8000.0,
                         "kernel": "k_stream_soa_vec<float,false,true>",
                         "bytes_per_particle": bpp},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "clocks": clk,
            "gpu_launches": 2 * args.steps,
            "diag_last_step": {"kinetic_energy_erg": final_diag[0], "count": final_diag[1]},
        }
        print(json.dumps(line), flush=True)
    ens.close()
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
