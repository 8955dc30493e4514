"""Seeded synthetic inputs for the Boris push -- shared by tests and bench.

This module holds NONE of the method's arithmetic (no Boris step, no field
formula, no kinetic energy).  It only draws reproducible random numbers with a
counter-based hash (value = f(seed, stream, global particle index)), so that

* the same particle gets the same values on CPU and GPU, in any shard and in
  any chunking (sharded == unsharded, bit for bit, on one device);
* inputs for 8e8 particles can be generated chunk by chunk on the device.

Workload recipes follow the paper's benchmark shape (PAPER.md
L427-434: electrons at rest, uniform in a sphere of radius 0.6 lambda,
lambda = 0.9 um, omega0 = 2.1e15 s^-1) and BASELINE.json's five configs.
Units are Gaussian CGS (reading c1).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import torch

# CODATA 2018, Gaussian CGS (SURVEY §8(c) reading c1).
E_CHARGE = 4.80320471e-10        # statC
M_ELECTRON = 9.1093837015e-28    # g
M_PROTON = 1.67262192369e-24     # g
C_LIGHT = 29979245800.0          # cm/s
OMEGA0 = 2.1e15                  # s^-1
LAMBDA0 = 2.0 * math.pi * C_LIGHT / OMEGA0   # 0.897 um (L414: "0.9 um")
T0 = 2.0 * math.pi / OMEGA0      # laser period
SPHERE_RADIUS = 0.6 * LAMBDA0
E_UNIT = M_ELECTRON * C_LIGHT * OMEGA0 / E_CHARGE   # relativistic field unit m c w0 / e

ELECTRON = (-E_CHARGE, M_ELECTRON)
POSITRON = (+E_CHARGE, M_ELECTRON)
PROTON = (+E_CHARGE, M_PROTON)

_MASK32 = 0xFFFFFFFF
_M1 = 0x045D9F3B   # < 2^31, so a 32x27-bit product never overflows int64


def _mix32(x: torch.Tensor) -> torch.Tensor:
    """A 32-bit integer finaliser on int64 tensors holding values in [0, 2^32)."""
    x = x ^ (x >> 16)
    x = (x * _M1) & _MASK32
    x = x ^ (x >> 16)
    x = (x * _M1) & _MASK32
    x = x ^ (x >> 16)
    return x


def hash_u32(seed: int, stream: int, idx: torch.Tensor) -> torch.Tensor:
    """Counter-based 32-bit hash of (seed, stream, idx) -> int64 in [0, 2^32)."""
    key = _mix32(torch.tensor(((seed * 7919 + stream * 104729) & _MASK32), dtype=torch.int64,
                              device=idx.device))
    lo = idx & _MASK32
    hi = idx >> 32
    h = _mix32(lo ^ key)
    h = _mix32((h + hi * 0x3C6EF372 + stream) & _MASK32)
    return _mix32(h ^ key)


def uniform(seed: int, stream: int, idx: torch.Tensor) -> torch.Tensor:
    """float64 uniform in the open interval (0, 1)."""
    return (hash_u32(seed, stream, idx).to(torch.float64) + 0.5) * (1.0 / 4294967296.0)


def normal(seed: int, stream: int, idx: torch.Tensor) -> torch.Tensor:
    """float64 standard normal (Box-Muller on two hashed uniforms)."""
    u1 = uniform(seed, 2 * stream + 1000, idx)
    u2 = uniform(seed, 2 * stream + 1001, idx)
    return torch.sqrt(-2.0 * torch.log(u1)) * torch.cos(2.0 * math.pi * u2)


def in_sphere(seed: int, idx: torch.Tensor, radius: float):
    """Uniform points in a ball (L427-428): radius R u^{1/3}, isotropic direction."""
    rr = radius * uniform(seed, 1, idx).pow(1.0 / 3.0)
    cos_t = 1.0 - 2.0 * uniform(seed, 2, idx)
    sin_t = torch.sqrt(torch.clamp(1.0 - cos_t * cos_t, min=0.0))
    ph = 2.0 * math.pi * uniform(seed, 3, idx)
    return rr * sin_t * torch.cos(ph), rr * sin_t * torch.sin(ph), rr * cos_t


def isotropic(seed: int, idx: torch.Tensor, magnitude: float, stream0: int = 10):
    cos_t = 1.0 - 2.0 * uniform(seed, stream0, idx)
    sin_t = torch.sqrt(torch.clamp(1.0 - cos_t * cos_t, min=0.0))
    ph = 2.0 * math.pi * uniform(seed, stream0 + 1, idx)
    return magnitude * sin_t * torch.cos(ph), magnitude * sin_t * torch.sin(ph), magnitude * cos_t


@dataclass
class Workload:
    """A synthetic ensemble recipe.  All values float64 / CGS unless noted."""
    name: str
    n: int
    seed: int
    types: list                     # [(charge, mass), ...]
    dt: float
    n_steps: int
    precision: str = "fp32"         # "fp32" | "fp64"
    layout: str = "soa"             # "soa" | "aos"
    field_kind: str = "arrays"      # "arrays" | "uniform" | "plane_wave"
    uniform_E: tuple = (0.0, 0.0, 0.0)
    uniform_B: tuple = (0.0, 0.0, 0.0)
    plane_wave: dict = field(default_factory=dict)
    field_sigma: float = 0.0        # per-particle E/B: Gaussian sigma per component
    mom_kind: str = "rest"          # "rest" | "gauss" | "shell"
    mom_scale: float = 0.0          # sigma (gauss) or |p| (shell)
    type_mix: str = "single"        # "single" | "random" (i.i.d. uniform over types)
    weight_kind: str = "one"        # "one" | "uniform"  (hash-uniform in [0.5, 1.5])
    light_velocity: float = C_LIGHT

    def generate(self, first: int = 0, count: int | None = None, device="cpu"):
        """Particles [first, first+count) of this workload as float64 tensors.

        Returns dict with x,y,z,px,py,pz,weight (float64), type (int16) and, for
        field_kind == "arrays", Ex..Bz (float64).  Values depend only on
        (seed, global index), never on `first`/`count` chunking.
        """
        if count is None:
            count = self.n - first
        return self.generate_indices(
            torch.arange(first, first + count, dtype=torch.int64, device=device))

    def generate_indices(self, idx: torch.Tensor):
        """The particles with the given global indices (int64 tensor), as generate()."""
        device = idx.device
        count = idx.numel()
        out = {}
        out["x"], out["y"], out["z"] = in_sphere(self.seed, idx, SPHERE_RADIUS)
        if self.mom_kind == "rest":
            z = torch.zeros(count, dtype=torch.float64, device=device)
            out["px"], out["py"], out["pz"] = z, z.clone(), z.clone()
        elif self.mom_kind == "gauss":
            out["px"] = self.mom_scale * normal(self.seed, 20, idx)
            out["py"] = self.mom_scale * normal(self.seed, 21, idx)
            out["pz"] = self.mom_scale * normal(self.seed, 22, idx)
        elif self.mom_kind == "shell":
            out["px"], out["py"], out["pz"] = isotropic(self.seed, idx, self.mom_scale)
        else:
            raise ValueError(self.mom_kind)
        if self.weight_kind == "one":
            out["weight"] = torch.ones(count, dtype=torch.float64, device=device)
        else:
            out["weight"] = 0.5 + uniform(self.seed, 30, idx)
        if self.type_mix == "single" or len(self.types) == 1:
            out["type"] = torch.zeros(count, dtype=torch.int16, device=device)
        else:
            out["type"] = (hash_u32(self.seed, 31, idx) % len(self.types)).to(torch.int16)
        if self.field_kind == "arrays":
            for j, comp in enumerate(("Ex", "Ey", "Ez", "Bx", "By", "Bz")):
                out[comp] = self.field_sigma * normal(self.seed, 40 + j, idx)
        return out


def gyro_period(q: float, m: float, B: float, gamma: float, c: float = C_LIGHT) -> float:
    """T = 2 pi gamma m c / (|q| B) -- workload sizing only (sets dt)."""
    return 2.0 * math.pi * gamma * m * c / (abs(q) * B)


B0 = M_ELECTRON * C_LIGHT * OMEGA0 / E_CHARGE   # B with omega_c(gamma=1) = omega0


def config(name: str, n: int | None = None) -> Workload:
    """BASELINE.json configs[0..4] as synthetic recipes."""
    if name == "C1":
        # 1000 e-, uniform B, |p| = m c (gamma0 = sqrt 2), dt = 0.01 T_gyro, 100 steps.
        tg = gyro_period(E_CHARGE, M_ELECTRON, B0, math.sqrt(2.0))
        return Workload("C1", n or 1000, 1, [ELECTRON], 0.01 * tg, 100, "fp64", "soa",
                        "uniform", uniform_B=(0.0, 0.0, B0), mom_kind="shell",
                        mom_scale=M_ELECTRON * C_LIGHT)
    if name == "C2":
        # 1e7, per-particle E/B (sigma = 80 m c w0/e per component), dt = T/1e4, 1 step/launch.
        return Workload("C2", n or 10_000_000, 2, [ELECTRON], T0 / 1.0e4, 1, "fp32", "soa",
                        "arrays", field_sigma=80.0 * E_UNIT, mom_kind="gauss",
                        mom_scale=M_ELECTRON * C_LIGHT)
    if name == "C3":
        # 1e7, e-/e+/p random types, crossed E x B (E = 0.5 B), at rest, dt = T_lab,e/100.
        gd = 2.0 / math.sqrt(3.0)
        tl = 2.0 * math.pi * gd ** 3 * M_ELECTRON * C_LIGHT / (E_CHARGE * B0)
        return Workload("C3", n or 10_000_000, 3, [ELECTRON, POSITRON, PROTON], tl / 100.0, 100,
                        "fp64", "aos", "uniform", uniform_E=(0.0, 0.5 * B0, 0.0),
                        uniform_B=(0.0, 0.0, B0), type_mix="random")
    if name == "C4":
        # 1e8 e- at rest, plane wave k=x, e=y, a0 = 10, dt = T/100, 100 steps fused.
        return Workload("C4", n or 100_000_000, 4, [ELECTRON], T0 / 100.0, 100, "fp32", "soa",
                        "plane_wave",
                        plane_wave=dict(E0=10.0 * E_UNIT, k_hat=(1.0, 0.0, 0.0),
                                        e_hat=(0.0, 1.0, 0.0), omega=OMEGA0,
                                        k=OMEGA0 / C_LIGHT, phase0=0.0))
    if name == "C5":
        # 8e8 total, C2 recipe by global index, weights in [0.5, 1.5], per-step KE.
        return Workload("C5", n or 800_000_000, 5, [ELECTRON], T0 / 1.0e4, 1, "fp32", "soa",
                        "arrays", field_sigma=80.0 * E_UNIT, mom_kind="gauss",
                        mom_scale=M_ELECTRON * C_LIGHT, weight_kind="uniform")
    raise ValueError(name)

