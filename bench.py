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
# The bench always times boris_push_diag (the KE diagnostic reads the 4 B weight), so C2
# through this path also moves 80 B; the 76 B C2 figure belongs to boris_push without the
# diagnostic (the "configs" entries below).
BYTES_PER_PARTICLE_STEP = {"C5": 80, "C2": 80}
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


def host_cpu():
    """The host CPU the oracle ran on (model, logical CPUs, affinity, OpenMP binding)."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        affinity = len(os.sched_getaffinity(0))
    except Exception:
        affinity = None
    return {"model": model, "logical_cpus": os.cpu_count(), "affinity_cpus": affinity,
            "omp_proc_bind": os.environ.get("OMP_PROC_BIND"),
            "omp_places": os.environ.get("OMP_PLACES")}


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
            "kind": "oracle", "host": host_cpu(),
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


ALU_COUNTS = os.path.join(ROOT, "profiles", "alu_counts.json")


def alu_bound_ps(kernel_key, sm_mhz):
    """Lower bound (ps per particle-step) of a register-fused kernel from its ncu-measured
    executed warp-instructions per warp-step (profiles/alu_counts.json) and the B200 unit
    counts: issue 1 warp-instruction/clk per SMSP (4 per SM), XU (MUFU)
    16 lanes/clk/SM, FP64 64 lanes/clk/SM; 148 SMs.  Returns (bound_ps, limiter) or None."""
    try:
        ent = json.load(open(ALU_COUNTS))["kernels"][kernel_key]
    except Exception:
        return None
    f = sm_mhz * 1e6
    sms = 148
    per_ws = {"issue": ent["inst_per_warp_step"] / (4 * sms * f) / 32,
              "xu": ent["xu_per_warp_step"] * 32 / (16 * sms * f) / 32,
              "fp64": ent["fp64_per_warp_step"] * 32 / (64 * sms * f) / 32}
    lim = max(per_ws, key=per_ws.get)
    return per_ws[lim] * 1e12, lim


def _time_launches(torch, fn, iters, warmup=2):
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


def measure_configs(torch, synth, lb, peak, sm_max_mhz):
    """Every BASELINE.json config on this GPU, measured in the same run as the headline
    (rank 0, N=1): the streaming ones against the HBM roofline (algorithmic / layout-
    implied bytes), the register-fused ones against the ALU roofline."""
    from paper_2104_04579_b200.ensemble import AosEnsemble, SoaEnsemble
    import numpy as np
    PREC = {"fp32": lb.BORIS_FP32, "fp64": lb.BORIS_FP64}
    sp = torch.cuda.current_stream().cuda_stream
    out = {}

    def make(w, layout, precision, n, field_kind=None):
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
            field = lb.boris_field_create_plane_wave(pw["E0"], pw["k_hat"], pw["e_hat"],
                                                     pw["omega"], pw["k"], pw["phase0"])
        else:
            md = w.plane_wave
            field = lb.boris_field_create_mdipole(md["A0"], md["omega0"], md["k"])
        torch.cuda.synchronize()
        return ens, field

    def streaming(key, layout, precision, n, iters=20):
        w = synth.config("C2", n=n)
        ens, field = make(w, layout, precision, n)
        fs = 4 if precision == "fp32" else 8
        alg = 19 * fs                                   # R r,p,E,B; W r,p,gamma
        bpp = alg if layout == "soa" else (36 if fs == 4 else 72) * 2 + 6 * fs
        ms = _time_launches(torch, lambda: lb.boris_push(ens.handle, field, w.dt, 1, sp), iters)
        ens.close()
        gbs = bpp * n / (ms * 1e-3) / 1e9
        out[key] = {"workload": f"C2 (BASELINE configs[1]) {layout.upper()} {precision}, "
                                f"per-particle E/B, 1 step per launch, boris_push",
                    "n": n, "ms_per_launch": ms, "ps_per_particle_step": ms * 1e9 / n,
                    "particle_updates_per_s": n / (ms * 1e-3),
                    "roofline": {"bound": "hbm", "achieved": gbs, "peak": peak, "unit": "GB/s",
                                 "frac": gbs / peak, "frac_of_nominal_8tbs": gbs / 8000.0,
                                 "bytes_per_particle": bpp,
                                 "bytes_kind": "algorithmic" if layout == "soa"
                                 else f"layout-implied (algorithmic {alg})"}}

    def fused(key, cfg, layout, precision, n, steps, kernel_key, iters=5, mdipole=False,
              label=None):
        w = synth.config(cfg, n=n)
        if mdipole:
            # 1e7 e- at rest in the 0.6-lambda sphere, m-dipole 0.1 PW
            # (reading c12), dt = T/1e4 (c7), 1e3 steps per iteration
            k = synth.OMEGA0 / synth.C_LIGHT
            w.field_kind = "mdipole"
            w.plane_wave = dict(A0=k * math.sqrt(3e21 / synth.C_LIGHT), omega0=synth.OMEGA0, k=k)
            w.dt = synth.T0 / 1e4
        ens, field = make(w, layout, precision, n)
        ms = _time_launches(torch, lambda: lb.boris_push(ens.handle, field, w.dt, steps, sp),
                            iters, warmup=1)
        ens.close()
        lb.boris_field_destroy(field)
        ps = ms * 1e9 / (n * steps)
        ent = {"workload": label, "n": n, "steps_per_launch": steps, "ms_per_launch": ms,
               "ps_per_particle_step": ps, "particle_updates_per_s": 1e12 / ps}
        b = alu_bound_ps(kernel_key, sm_max_mhz)
        if b is not None:
            ent["roofline"] = {"bound": "alu", "achieved": 1e12 / ps, "peak": 1e12 / b[0],
                               "unit": "particle-updates/s", "frac": b[0] / ps,
                               "limiter": b[1], "bound_ps_per_particle_step": b[0],
                               "kernel": kernel_key}
        if mdipole:
            ent["nsps"] = ps * 1e-3     # the paper's ns per particle per step (Table 2)
        out[key] = ent

    t0 = time.perf_counter()
    # configs[0] (C1): closed-form Larmor check of the fp64 fused kernel, 100 steps
    out["C1"] = c1_closed_form(torch, synth, lb, np)
    # configs[1] (C2): 1e7, all four layout x precision cells; plus the north_star size 1e8
    streaming("C2_soa_fp32_1e8", "soa", "fp32", 100_000_000)
    for layout in ("soa", "aos"):
        for prec in ("fp32", "fp64"):
            streaming(f"C2_{layout}_{prec}_1e7", layout, prec, 10_000_000)
    # configs[2] (C3), configs[3] (C4): register-fused, 100 steps per launch
    fused("C3_aos_fp64", "C3", "aos", "fp64", 10_000_000, 100, "C3_aos_fp64_uniform_yz",
          label="C3 (configs[2]): 1e7, e-/e+/p, crossed ExB, fp64 AoS, 100 fused steps")
    fused("C4_soa_fp32", "C4", "soa", "fp32", 100_000_000, 100, "C4_soa_fp32_planewave_yz",
          label="C4 (configs[3]): 1e8, plane wave a0=10, fp32 SoA, 100 fused steps")
    # the paper's analytic Table-2 cells (m-dipole 0.1 PW, 1e7 e-, 1e3 steps per iteration)
    for layout in ("soa", "aos"):
        for prec in ("fp32", "fp64"):
            fused(f"table2_analytic_{layout}_{prec}", "C4", layout, prec, 10_000_000, 1000,
                  f"mdipole_{layout}_{prec}", iters=2, mdipole=True,
                  label=f"PAPER Table 2 analytic cell {layout.upper()} {prec}: 1e7 e- at rest "
                        f"in 0.6 lambda, m-dipole 0.1 PW, 1e3 fused steps")
    out["wall_s"] = time.perf_counter() - t0
    return out


def c1_closed_form(torch, synth, lb, np):
    """BASELINE configs[0]: 1000 e-, uniform B, |p| = mc, dt = 0.01 T_gyro, 100 steps, fp64
    SoA, vs the discrete Larmor closed form: u_perp rotates by
    alpha = -2 atan(t_z) per step, r^N = r^0 + (c dt/gamma) sum_n R(n alpha) u_perp^0."""
    from paper_2104_04579_b200.ensemble import SoaEnsemble
    w = synth.config("C1")
    d = w.generate()
    ens = SoaEnsemble(w.n, lb.BORIS_FP64, w.types, w.light_velocity, with_fields=False)
    ens.fill(d)
    ens.wrap()
    field = lb.boris_field_create_uniform(w.uniform_E, w.uniform_B)
    lb.boris_push(ens.handle, field, w.dt, w.n_steps, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    s = {k: ens.t[k].cpu().numpy() for k in ("x", "y", "z", "px", "py", "pz")}
    lb.boris_field_destroy(field)
    ens.close()
    q, m = w.types[0]
    c, B, N = w.light_velocity, w.uniform_B[2], w.n_steps
    gamma = math.sqrt(2.0)
    alpha = -2 * math.atan(q * B * w.dt / (2 * gamma * m * c))
    u0 = np.stack([d["px"].numpy(), d["py"].numpy(), d["pz"].numpy()], 1) / (m * c)
    z0 = u0[:, 0] + 1j * u0[:, 1]
    e = np.exp(1j * alpha)
    zN = z0 * np.exp(1j * N * alpha)
    sm = z0 * e * (1 - np.exp(1j * N * alpha)) / (1 - e)
    cdt = c * w.dt / gamma
    r_ref = np.stack([d["x"].numpy() + cdt * sm.real, d["y"].numpy() + cdt * sm.imag,
                      d["z"].numpy() + N * cdt * u0[:, 2]], 1)
    u_ref = np.stack([zN.real, zN.imag, u0[:, 2]], 1)
    p_err = float(np.abs(np.stack([s["px"], s["py"], s["pz"]], 1) / (m * c) - u_ref).max())
    r_err = float(np.abs(np.stack([s["x"], s["y"], s["z"]], 1) - r_ref).max() / (c * w.dt))
    return {"workload": "C1 (configs[0]): 1000 e-, uniform B, fp64 SoA, dt = 0.01 T_gyro, "
                        "100 steps, vs the discrete Larmor closed form",
            "p_err_over_mc": p_err, "r_err_over_c_dt": r_err,
            "pass": bool(p_err < 1e-12 and r_err < 1e-10)}


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
                         "host": host_cpu(),
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
    ap.add_argument("--no-configs", action="store_true",
                    help="skip the per-BASELINE-config measurements (N=1 only)")
    args = ap.parse_args()
    if int(os.environ.get("WORLD_SIZE", 1)) > 1:
        # NCCL's INIT lines (communicator size, NVLS / P2P transport) for the driver's log
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
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
    n_local_max = int(bdist.max_over_ranks(float(n_local), dev))
    final_diag = diag[(args.steps - 1) % 2].tolist()
    # the allreduced count of the last timed step must be the whole ensemble (every rank's
    # push and the NCCL sum took part); anything else is a failed run, not a number
    if final_diag[1] != float(w.n):
        raise SystemExit(f"bench: diagnostic count {final_diag[1]} != {w.n} particles "
                         f"(rank {rank}/{world})")

    ms_per_step = elapsed_ms / args.steps
    value = w.n * args.steps / (elapsed_ms * 1e-3)            # whole-job particle-updates/s
    peak, peak_kind = measured_peak()
    # GB/s of the push kernel on the slowest rank (largest shard, max push time over ranks)
    achieved = bpp * n_local_max / (push_ms_max * 1e-3) / 1e9
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

    configs = None
    if rank == 0 and world == 1 and not args.no_configs:
        ens.close()
        ens = None                      # free the C5 arrays before the config ensembles
        torch.cuda.empty_cache()
        try:
            sm_max = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
                           .get("sm_max_mhz", 1965.0))
        except Exception:
            sm_max = 1965.0
        configs = measure_configs(torch, synth, lb, peak, sm_max)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "particle-updates/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "ns_per_particle_step": 1e9 / value,
            "hbm_gbs_per_gpu": achieved,
            "push_ms_max_over_ranks": push_ms_max, "particles_per_gpu_max": n_local_max,
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
            "baseline_configs": configs,
        }
        print(json.dumps(line), flush=True)
    if ens is not None:
        ens.close()
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
