"""Shared helpers for GPU <-> oracle parity tests (test infrastructure)."""
from __future__ import annotations

import numpy as np
import torch

import oracle

# Tolerances from BASELINE.json north_star: "relative error <= 1e-12 for fp64 and
# <= 1e-5 for fp32 after 100 steps", with the metric of reading c15.
TOL = {"fp64": 1e-12, "fp32": 1e-5}


class C15:
    """Reading c15: per particle ||x_gpu - x_ref|| / (||x_ref|| + S_x), with S_x the
    trajectory scale max_{s' <= s} rms_j ||x_ref,j(s')||."""

    def __init__(self):
        self.scale = {}

    def __call__(self, key, gpu, ref):
        nrm = np.linalg.norm(ref, axis=1)
        self.scale.setdefault(key, 0.0)
        if nrm.size:
            self.scale[key] = max(self.scale[key], float(np.sqrt(np.mean(nrm ** 2))))
        s = self.scale[key] if self.scale[key] > 0 else 1.0
        err = np.linalg.norm(gpu - ref, axis=1) / (nrm + s)
        return float(err.max()) if err.size else 0.0


def rounded(d, precision):
    """The generator's float64 values rounded to the kernel's storage precision (the
    oracle starts from the same rounded inputs, reading c15)."""
    dt = torch.float32 if precision == "fp32" else torch.float64
    out = {}
    for k, v in d.items():
        out[k] = v.to(dt).to(torch.float64) if v.dtype == torch.float64 else v.clone()
    return out


def stack3(d, a, b, c):
    return torch.stack([d[a], d[b], d[c]], 1).numpy().astype(np.float64)


def oracle_field(w, precision, xi=None):
    """Oracle (kind, params) for a synth.Workload's analytic field."""
    if w.field_kind == "uniform":
        return oracle.FIELD_UNIFORM, list(w.uniform_E) + list(w.uniform_B)
    if w.field_kind == "plane_wave":
        pw = w.plane_wave
        return oracle.FIELD_PLANE_WAVE, ([pw["E0"]] + list(pw["k_hat"]) + list(pw["e_hat"]) +
                                         [pw["omega"], pw["k"], pw["phase0"]])
    if w.field_kind == "mdipole":
        md = w.plane_wave  # reuse dict slot: A0, omega0, k
        xs, nt = (1.0, 9) if precision == "fp64" else (1.5, 7)
        return oracle.FIELD_MDIPOLE, [md["A0"], md["omega0"], md["k"], xs, nt]
    return oracle.FIELD_ARRAYS, None


class OracleRun:
    """The oracle's state for one workload, advanced in chunks like the GPU."""

    def __init__(self, w, d, precision, pusher=0):
        self.pusher = pusher
        self.w = w
        self.pos = stack3(d, "x", "y", "z")
        self.mom = stack3(d, "px", "py", "pz")
        self.type = d["type"].numpy().astype(np.int16)
        self.weight = d["weight"].numpy().astype(np.float64)
        self.tq = [q for q, m in w.types]
        self.tm = [m for q, m in w.types]
        self.kind, self.params = oracle_field(w, precision)
        if self.kind == oracle.FIELD_ARRAYS:
            self.E = stack3(d, "Ex", "Ey", "Ez")
            self.B = stack3(d, "Bx", "By", "Bz")
        else:
            self.E = self.B = None
        self.t = 0.0
        self.gamma = None

    def push(self, n_steps):
        self.pos, self.mom, self.gamma = oracle.push(
            self.pos, self.mom, self.type, self.tq, self.tm, self.w.light_velocity, self.kind,
            self.params, E=self.E, B=self.B, t0=self.t, dt=self.w.dt, n_steps=n_steps,
            pusher=self.pusher)
        self.t += n_steps * self.w.dt

    def kinetic_energy(self):
        return oracle.kinetic_energy(self.mom, self.gamma, self.weight, self.type, self.tm,
                                     self.w.light_velocity)


# Unit roundoff of the storage precision: a stored position is fl(r) = r (1 + d), |d| <= u.
UNIT_ROUNDOFF = {"fp32": 2.0 ** -24, "fp64": 2.0 ** -53}


class Displacement:
    """Reading c15 applied to the displacement dr = r - r0 (eq. 7: the position
    update is the only place dt/(gamma m) enters r), both sides from the same rounded r0.

    The c15 position metric is floored at the trajectory scale rms|r| (~0.47 lambda in
    C2/C5), while one C2 step moves a particle by <= c dt = lambda/1e4, so an error in
    a10 of ~5 % of a step would hide under it.  Two checks on dr instead:

    * per particle: |dr_gpu - dr_ref| - A <= tol (|dr_ref| + S_dr), S_dr the trajectory
      scale of dr (max over checks of rms|dr_ref|), and A = n_stores u (|r0| + |r_ref| +
      |dr_ref|) the rounding of the n_stores positions the kernel stored in FP since r0
      (each fl(r^n) errs by <= u |r^n|; |r^n| <= |r0| + path).  A is what any FP-storage
      implementation incurs; for fp32 single steps it dominates;
    * ensemble bias: b = sum_i (dr_gpu - dr_ref).dr_ref / sum_i |dr_ref|^2, the relative
      scale error of the GPU's displacements.  Storage rounding does not average to zero
      exactly: each particle contributes at most A_i |dr_i| to the numerator with an
      input-dependent sign, so b carries rounding noise up to
      N_b = 5 sqrt(sum_i (A_i |dr_i|)^2) / sum_i |dr_i|^2 (5 sigma for independent
      signs; it matters when |dr| is a few ulp of |r|, e.g. particles 2 steps from rest).
      A systematic error in a10 (e.g. a wrong dt/(S m)) does not average out:
      |b| - N_b <= tol.  The second value returned is sign(b) max(|b| - N_b, 0).
    """

    def __init__(self, r0, precision):
        self.r0 = np.array(r0, dtype=np.float64, copy=True)
        self.u = UNIT_ROUNDOFF[precision]
        self.scale = 0.0

    def __call__(self, r_gpu, r_ref, n_stores, idx=None):
        r0 = self.r0 if idx is None else self.r0[idx]
        dg = r_gpu - r0
        dr = r_ref - r0
        nrm = np.linalg.norm(dr, axis=1)
        if nrm.size:
            self.scale = max(self.scale, float(np.sqrt(np.mean(nrm ** 2))))
        s = self.scale if self.scale > 0 else 1.0
        allow = n_stores * self.u * (np.linalg.norm(r0, axis=1) + np.linalg.norm(r_ref, axis=1)
                                     + nrm)
        diff = dg - dr
        err = np.maximum(np.linalg.norm(diff, axis=1) - allow, 0.0) / (nrm + s)
        den = float(np.sum(dr * dr))
        bias = float(np.sum(diff * dr)) / den if den > 0 else 0.0
        noise = 5.0 * float(np.sqrt(np.sum((allow * nrm) ** 2))) / den if den > 0 else 0.0
        self.last_bias, self.last_noise = bias, noise
        excess = np.sign(bias) * max(abs(bias) - noise, 0.0)
        return (float(err.max()) if err.size else 0.0), float(excess)
