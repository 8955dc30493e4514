"""Boris-push oracle -- TEST INFRASTRUCTURE ONLY.

A plain, slow, scalar double-precision CPU implementation of the relativistic
Boris push of arXiv 2104.04579 §2, written in C
(``oracle/boris_oracle.c``) and loaded here with ctypes.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  It shares no code with the
CUDA path (``paper_2104_04579_b200``) and never imports it.

Arrays are numpy, canonical double, xyz-interleaved (``pos``/``mom`` are
``(n, 3)``).  Field kinds and parameter vectors are the oracle's own:

* ``FIELD_ARRAYS``      per-particle ``E``/``B`` ``(n, 3)``, constant over steps (L369-371)
* ``FIELD_UNIFORM``     params ``[Ex, Ey, Ez, Bx, By, Bz]``
* ``FIELD_PLANE_WAVE``  params ``[E0, kx, ky, kz, ex, ey, ez, omega, k, phase0]``
* ``FIELD_MDIPOLE``     params ``[A0, omega0, k, xi_star, n_terms]`` (eq. 14-15, readings c9-c13)
* ``FIELD_GRID``        params ``[x0, y0, z0, dx, dy, dz, nx, ny, nz]``; ``E``/``B`` = node values
  ``(3, nz, ny, nx)``, CIC gather on a periodic collocated grid (reading c-grid)

Pins: ``tests/test_oracle_pins.py`` (closed forms, invariants, hand cases).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

FIELD_ARRAYS = 0
FIELD_UNIFORM = 1
FIELD_PLANE_WAVE = 2
FIELD_MDIPOLE = 3
FIELD_GRID = 4

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "boris_oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

_dp = ctypes.POINTER(ctypes.c_double)
_i16p = ctypes.POINTER(ctypes.c_int16)


def build(force: bool = False) -> str:
    """Compile ``liboracle.so`` with gcc (-O2, no -ffast-math, OpenMP driver)."""
    if force or not os.path.exists(_LIB_PATH) or (
        os.path.getmtime(_LIB_PATH) < max(os.path.getmtime(_SRC),
                                           os.path.getmtime(os.path.join(_HERE, "boris_oracle.h")))
    ):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        # -ffp-contract=off: the oracle rounds every operation as written (reading c14
        # allows contraction on either side; the oracle takes the plain reading).
        cmd = ["gcc", "-std=c11", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
               "-fPIC", "-shared", "-o", tmp, _SRC, "-lm"]
        subprocess.check_call(cmd)
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB_PATH)
        lib.oracle_boris_step.argtypes = [_dp, _dp, _dp, ctypes.c_double, ctypes.c_double,
                                          ctypes.c_double, _dp, _dp, ctypes.c_double]
        lib.oracle_boris_step.restype = None
        lib.oracle_field_plane_wave.argtypes = [_dp, _dp, ctypes.c_double, _dp, _dp]
        lib.oracle_field_mdipole.argtypes = [_dp, _dp, ctypes.c_double, _dp, _dp]
        lib.oracle_field_grid.argtypes = [_dp, _dp, _dp, _dp, _dp, _dp]
        lib.oracle_mdipole_radial.argtypes = [ctypes.c_double, ctypes.c_double, ctypes.c_int,
                                              _dp, _dp, _dp]
        lib.oracle_push.argtypes = [ctypes.c_int64, _dp, _dp, _dp, _i16p, _dp, _dp,
                                    ctypes.c_int32, ctypes.c_double, ctypes.c_int, _dp, _dp, _dp,
                                    ctypes.c_double, ctypes.c_double, ctypes.c_int64, ctypes.c_int]
        lib.oracle_push.restype = ctypes.c_int
        lib.oracle_kinetic_energy.argtypes = [ctypes.c_int64, _dp, _dp, _dp, _i16p, _dp,
                                              ctypes.c_double]
        lib.oracle_kinetic_energy.restype = ctypes.c_double
        lib.oracle_neumaier_sum.argtypes = [ctypes.c_int64, _dp]
        lib.oracle_neumaier_sum.restype = ctypes.c_double
        lib.oracle_max_threads.restype = ctypes.c_int
        for name in ("oracle_vay_step", "oracle_hc_step"):
            getattr(lib, name).argtypes = lib.oracle_boris_step.argtypes
            getattr(lib, name).restype = None
        lib.oracle_set_pusher.argtypes = [ctypes.c_int]
        lib.oracle_deposit_current.argtypes = [ctypes.c_int64, _dp, _dp, _dp, _i16p, _dp, _dp,
                                               ctypes.c_double, ctypes.c_double, _dp, _dp]
        lib.oracle_deposit_current.restype = None
        _lib = lib
    return _lib


def _d(a):
    return a.ctypes.data_as(_dp)


def _f64(a, shape=None):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    if shape is not None:
        a = a.reshape(shape)
    return a


PUSHER_BORIS = 0
PUSHER_VAY = 1
PUSHER_HIGUERA_CARY = 2


def boris_step(r, p, q, m, c, E, B, dt, pusher=PUSHER_BORIS):
    """One step of one particle (Boris: L175-186; Vay / Higuera-Cary: readings c-vay,
    c-hc).  Returns (r_new, p_new, gamma)."""
    lib = _load()
    r = _f64(r, (3,)).copy()
    p = _f64(p, (3,)).copy()
    g = np.zeros(1)
    fn = {PUSHER_BORIS: lib.oracle_boris_step, PUSHER_VAY: lib.oracle_vay_step,
          PUSHER_HIGUERA_CARY: lib.oracle_hc_step}[pusher]
    fn(_d(r), _d(p), _d(g), q, m, c, _d(_f64(E, (3,))), _d(_f64(B, (3,))), dt)
    return r, p, float(g[0])


def push(pos, mom, type_, type_q, type_m, c, field_kind, params=None, E=None, B=None,
         t0=0.0, dt=1.0, n_steps=1, n_threads=1, pusher=PUSHER_BORIS):
    """Push copies of ``pos``/``mom`` ``n_steps`` steps.  Returns (pos, mom, gamma)."""
    lib = _load()
    lib.oracle_set_pusher(int(pusher))
    pos = _f64(pos).reshape(-1, 3).copy()
    mom = _f64(mom).reshape(-1, 3).copy()
    n = pos.shape[0]
    gamma = np.zeros(n)
    type_ = np.ascontiguousarray(np.asarray(type_, dtype=np.int16).reshape(n))
    tq = _f64(type_q).reshape(-1)
    tm = _f64(type_m).reshape(-1)
    params_a = _f64(params if params is not None else np.zeros(1)).reshape(-1)
    if field_kind == FIELD_ARRAYS:
        Ea = _f64(E).reshape(n, 3)
        Ba = _f64(B).reshape(n, 3)
        pE, pB = _d(Ea), _d(Ba)
    elif field_kind == FIELD_GRID:
        # E, B: node values, component-major (3, nz, ny, nx) -> flat
        Ea = _f64(E).reshape(-1)
        Ba = _f64(B).reshape(-1)
        pE, pB = _d(Ea), _d(Ba)
    else:
        pE = pB = ctypes.cast(None, _dp)
    rc = lib.oracle_push(n, _d(pos), _d(mom), _d(gamma), type_.ctypes.data_as(_i16p), _d(tq),
                         _d(tm), len(tq), c, field_kind, _d(params_a), pE, pB, t0, dt,
                         int(n_steps), int(n_threads))
    lib.oracle_set_pusher(PUSHER_BORIS)
    if rc != 0:
        raise ValueError("oracle_push: type index out of range")
    if n_steps == 0:
        gamma = np.sqrt(1.0 + np.sum(mom * mom, axis=1) / (tm[type_] * c) ** 2) if n else gamma
    return pos, mom, gamma


def kinetic_energy(mom, gamma, weight, type_, type_m, c):
    lib = _load()
    mom = _f64(mom).reshape(-1, 3)
    n = mom.shape[0]
    gamma = _f64(gamma).reshape(n)
    weight = _f64(weight).reshape(n)
    type_ = np.ascontiguousarray(np.asarray(type_, dtype=np.int16).reshape(n))
    tm = _f64(type_m).reshape(-1)
    return float(lib.oracle_kinetic_energy(n, _d(mom), _d(gamma), _d(weight),
                                           type_.ctypes.data_as(_i16p), _d(tm), c))


def neumaier_sum(x):
    lib = _load()
    x = _f64(x).reshape(-1)
    return float(lib.oracle_neumaier_sum(len(x), _d(x)))


def field_plane_wave(params, r, t):
    lib = _load()
    E = np.zeros(3)
    B = np.zeros(3)
    lib.oracle_field_plane_wave(_d(_f64(params)), _d(_f64(r, (3,))), t, _d(E), _d(B))
    return E, B


def field_grid(params, gridE, gridB, r):
    """CIC gather of node values (3, nz, ny, nx) at r (reading c-grid)."""
    lib = _load()
    E = np.zeros(3)
    B = np.zeros(3)
    gE = _f64(gridE).reshape(-1)
    gB = _f64(gridB).reshape(-1)
    lib.oracle_field_grid(_d(_f64(params)), _d(gE), _d(gB), _d(_f64(r, (3,))), _d(E), _d(B))
    return E, B


def deposit_current(pos, mom, weight, type_, type_q, type_m, c, dt, params):
    """Direct CIC current deposition at the half-step position (reading c-dep).
    pos/mom: state after the push.  Returns J as (3, nz, ny, nx)."""
    lib = _load()
    pos = _f64(pos).reshape(-1, 3)
    n = pos.shape[0]
    mom = _f64(mom).reshape(n, 3)
    weight = _f64(weight).reshape(n)
    type_ = np.ascontiguousarray(np.asarray(type_, dtype=np.int16).reshape(n))
    p = _f64(params).reshape(-1)
    nx, ny, nz = int(p[6]), int(p[7]), int(p[8])
    J = np.zeros((3, nz, ny, nx))
    lib.oracle_deposit_current(n, _d(pos), _d(mom), _d(weight), type_.ctypes.data_as(_i16p),
                               _d(_f64(type_q).reshape(-1)), _d(_f64(type_m).reshape(-1)), c, dt,
                               _d(p), _d(J))
    return J


def field_mdipole(params, r, t):
    lib = _load()
    E = np.zeros(3)
    B = np.zeros(3)
    lib.oracle_field_mdipole(_d(_f64(params)), _d(_f64(r, (3,))), t, _d(E), _d(B))
    return E, B


def mdipole_radial(xi, xi_star, n_terms):
    lib = _load()
    g1 = np.zeros(1)
    g2 = np.zeros(1)
    f3 = np.zeros(1)
    lib.oracle_mdipole_radial(xi, xi_star, int(n_terms), _d(g1), _d(g2), _d(f3))
    return float(g1[0]), float(g2[0]), float(f3[0])


def max_threads() -> int:
    return int(_load().oracle_max_threads())
