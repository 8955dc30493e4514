"""Pins of the oracle's DRIVER LOOP (``oracle_push``) for fields that depend on r or t.

``oracle_push`` (oracle/boris_oracle.c) samples the field at (r^n, t_n = t0 + n dt)
before every step (eq. 6 "E^n, B^n"; reading c5).  The pins in
``test_oracle_pins.py`` drive plane waves from a Python loop and grids only as a
constant, so the sampling inside ``oracle_push`` itself was unpinned.  Here every
physics check calls ``oracle.push`` directly, for runs that start at t0 != 0:

* plane wave (reading c-PW): the canonical momentum u_y + (qE0/mc w) sin(phi) and the
  light-front invariant gamma - u_x are exact constants of motion in a vacuum plane
  wave; Boris conserves them to O(dt^2);
* m-dipole (eq. 14, readings c9-c13): the field is axisymmetric with
  E = E_phi phi-hat, B_phi = 0, so A = A_phi phi-hat with E_phi = -(1/c) dA_phi/dt,
  A_phi = -(c/w0) 2 A0 k g1(kR) rho sin(w0 t), and the canonical angular momentum
  L_z = x p_y - y p_x + (q/c) rho A_phi
      = x p_y - y p_x - (2 q A0 k/w0) g1(kR) (x^2 + y^2) sin(w0 t)
  is exactly conserved (no phi dependence); Boris keeps it to O(dt^2);
* grid (reading c-grid): a periodic CIC grid holding E_x(x) (sampled sine) and a
  uniform B_z.  CIC makes E_x piecewise linear in x, whose potential phi(x) is the
  exact piecewise-quadratic integral of the node values, so gamma m c^2 + q phi(x) is
  exactly conserved (B does no work) and p_y + (q/c) B_z x too (no y dependence).

Each invariant is evaluated at the half step n+1/2 (p^{n+1/2}, x^{n+1/2} = (x^n +
x^{n+1})/2, t_{n+1/2}) against its value at n = -1/2 (p^{-1/2}, x^{-1/2} = x^0 - (dt/2)
v^{-1/2}, t0 - dt/2).  A pin passes when the drift is second order (ratio ~100 for a
10x smaller dt) and below an absolute bound.  ``test_pins_reject_mutated_sampling``
runs the SAME pins on explicit loops with the plausible driver mistakes (field at
t_{n+1/2}, at r^{n+1}, t0 ignored) and asserts that each mistake fails its pin; and
``test_driver_equals_explicit_loop`` ties ``oracle_push`` bitwise to the explicit
(r^n, t0 + n dt) loop.
"""
import math

import numpy as np
import pytest

import oracle

Q, M_, C = -1.0, 1.0, 1.0          # electron in normalised units (c = m = |q| = 1)
OMEGA = 1.0
T = 2 * math.pi / OMEGA
T0 = 0.37 * T                      # start time != 0 (reading c5: t_n = t0 + n dt)


# ---------------------------------------------------------------------------
# field set-ups
# ---------------------------------------------------------------------------

def _pw_params(a0=1.0, phase0=0.3):
    E0 = a0 * M_ * C * OMEGA / abs(Q)
    return [E0, 1, 0, 0, 0, 1, 0, OMEGA, OMEGA / C, phase0]


def _md_params(A0=1.0):
    return [A0, OMEGA, OMEGA / C, 1.0, 9]      # fp64 Taylor branch (c13): xi* = 1, 9 terms


GRID_NX, GRID_DX, GRID_X0 = 16, 0.5, -0.3
GRID_P = [GRID_X0, 0.1, -0.2, GRID_DX, 0.7, 0.9, GRID_NX, 3, 2]
GRID_E0, GRID_BZ, GRID_PH = 0.8, 0.6, 0.4


def _grid_nodes():
    nx, ny, nz = GRID_NX, 3, 2
    ex = GRID_E0 * np.sin(2 * np.pi * np.arange(nx) / nx + GRID_PH)
    gE = np.zeros((3, nz, ny, nx))
    gE[0] = ex[None, None, :]
    gB = np.zeros((3, nz, ny, nx))
    gB[2] = GRID_BZ
    return ex, gE, gB


def _grid_potential(x, ex):
    """phi(x) = -int_{x0}^{x} E_x dx for the CIC (piecewise-linear) interpolant of the node
    values ex: trapezoids over whole cells plus the partial cell, periodic images added as
    whole periods (the sine's period integral is ~0 but kept exactly)."""
    nx, dx = GRID_NX, GRID_DX
    cum = np.concatenate([[0.0], np.cumsum(0.5 * (ex + np.roll(ex, -1)) * dx)])
    xi = (x - GRID_X0) / dx
    i = np.floor(xi)
    f = xi - i
    ii = np.mod(i, nx).astype(int)
    per = np.floor(i / nx) * cum[nx]
    e0, e1 = ex[ii], ex[(ii + 1) % nx]
    return -(per + cum[ii] + dx * (e0 * f + (e1 - e0) * f * f / 2))


# ---------------------------------------------------------------------------
# invariants (evaluated at a half step)
# ---------------------------------------------------------------------------

def _gamma(p):
    return np.sqrt(1 + np.sum(p * p, -1) / (M_ * C) ** 2)


def _inv_plane_wave(params, xh, p, t):
    E0, k = params[0], params[8]
    u = p / (M_ * C)
    phi = k * xh[:, 0] - OMEGA * t + params[9]
    canon = u[:, 1] + Q * E0 / (M_ * C * OMEGA) * np.sin(phi)
    light_front = _gamma(p) - u[:, 0]
    return np.stack([canon, light_front], 1)


def _inv_mdipole(params, xh, p, t):
    A0, w0, k = params[0], params[1], params[2]
    x, y, z = xh[:, 0], xh[:, 1], xh[:, 2]
    R = np.sqrt(x * x + y * y + z * z)
    # g1 = f1/xi = j1(xi)/xi: scipy's spherical Bessel, not the oracle's own radial code
    import scipy.special
    xi = k * R
    g1 = np.where(xi > 1e-3, scipy.special.spherical_jn(1, np.maximum(xi, 1e-3)) /
                  np.maximum(xi, 1e-3), 1 / 3 - xi * xi / 30)
    Lz = x * p[:, 1] - y * p[:, 0] - (2 * Q * A0 * k / w0) * g1 * (x * x + y * y) * math.sin(w0 * t)
    return Lz[:, None]


def _inv_grid(ex, xh, p, t):
    H = _gamma(p) * M_ * C * C + Q * _grid_potential(xh[:, 0], ex)
    Py = p[:, 1] + Q / C * GRID_BZ * xh[:, 0]
    return np.stack([H, Py], 1)


# ---------------------------------------------------------------------------
# the pin: drift of the invariant from n = -1/2 to n = N/2 + 1/2 and N + 1/2
# ---------------------------------------------------------------------------

def _invariant_drift(push_n, inv, pos, mom, t0, dt, N):
    """max |I(n+1/2) - I(-1/2)| over n in {N/2, N}; push_n(k) -> state after k steps."""
    v = mom / (_gamma(mom) * M_)[:, None]
    I0 = inv(pos - 0.5 * dt * v, mom, t0 - 0.5 * dt)
    drift = 0.0
    for n in (N // 2, N):
        P1, _ = push_n(n)
        P2, M2 = push_n(n + 1)
        I = inv(0.5 * (P1 + P2), M2, t0 + (n + 0.5) * dt)
        drift = max(drift, float(np.abs(I - I0).max()))
    return drift


def _setup(kind):
    rng = np.random.default_rng({"pw": 41, "md": 42, "grid": 43}[kind])
    if kind == "pw":
        n = 8
        pos = np.c_[rng.uniform(-2, 2, n), rng.uniform(-1, 1, (n, 2))]
        mom = np.zeros((n, 3))
        params = _pw_params()
        field = (oracle.FIELD_PLANE_WAVE, params, None, None)
        inv = lambda xh, p, t: _inv_plane_wave(params, xh, p, t)
        fieldfn = lambda r, t: oracle.field_plane_wave(params, r, t)
    elif kind == "md":
        n = 8
        pos = rng.uniform(-1, 1, (n, 3)) * 2.5      # inside ~0.4 lambda: both radial branches
        mom = np.zeros((n, 3))
        params = _md_params()
        field = (oracle.FIELD_MDIPOLE, params, None, None)
        inv = lambda xh, p, t: _inv_mdipole(params, xh, p, t)
        fieldfn = lambda r, t: oracle.field_mdipole(params, r, t)
    else:
        n = 8
        pos = rng.uniform(-4, 4, (n, 3))
        mom = rng.normal(size=(n, 3)) * 0.7
        ex, gE, gB = _grid_nodes()
        field = (oracle.FIELD_GRID, GRID_P, gE, gB)
        inv = lambda xh, p, t: _inv_grid(ex, xh, p, t)
        fieldfn = lambda r, t: oracle.field_grid(GRID_P, gE, gB, r)
    return pos, mom, field, inv, fieldfn


def _driver_push(pos, mom, field, t0, dt):
    kind, params, E, B = field

    def push_n(k):
        P, Mo, _ = oracle.push(pos, mom, np.zeros(len(pos), np.int16), [Q], [M_], C, kind,
                               params, E=E, B=B, t0=t0, dt=dt, n_steps=k)
        return P, Mo
    return push_n


def _loop_push(pos, mom, fieldfn, t0, dt, mutation=None):
    """Explicit per-particle loop of oracle.boris_step with the field sampled at
    (r^n, t0 + n dt) -- or at a deliberately wrong place (``mutation``)."""
    def push_n(k):
        P, Mo = pos.copy(), mom.copy()
        for i in range(len(P)):
            r, p = P[i], Mo[i]
            for n in range(k):
                t, rs = t0 + n * dt, r
                if mutation == "t_half":
                    t = t + 0.5 * dt
                elif mutation == "t0_ignored":
                    t = n * dt
                elif mutation == "r_next":
                    rs = r + dt * p / (_gamma(p) * M_)
                E, B = fieldfn(rs, t)
                r, p, _ = oracle.boris_step(r, p, Q, M_, C, E, B, dt)
            P[i], Mo[i] = r, p
        return P, Mo
    return push_n


# absolute drift bounds at dt = T/1000 (measured 2.7e-6 .. 1.8e-6; mutated >= 1e-3)
BOUND = {"pw": 2e-5, "md": 2e-5, "grid": 2e-5}


def _pin(kind, make_push, steps=(100, 1000)):
    pos, mom, field, inv, fieldfn = _setup(kind)
    drifts = []
    for M in steps:
        dt = T / M
        drifts.append(_invariant_drift(make_push(pos, mom, field, fieldfn, dt), inv, pos, mom,
                                       T0, dt, M))
    return drifts


def _pin_ok(kind, drifts):
    # second order: ratio ~100 (grid: ~68, the CIC field has kinks at the nodes); first order ~10
    return 40 < drifts[0] / drifts[1] < 250 and drifts[1] < BOUND[kind]


@pytest.mark.parametrize("kind", ["pw", "md", "grid"])
def test_driver_conserves_exact_invariants_second_order(kind):
    drifts = _pin(kind, lambda pos, mom, field, fieldfn, dt: _driver_push(pos, mom, field, T0, dt))
    assert _pin_ok(kind, drifts), drifts


def test_plane_wave_driver_light_front_invariant_from_rest():
    """gamma - u_x = 1 for a particle that starts at rest (any phase, any t0)."""
    pos, mom, field, inv, _ = _setup("pw")
    dt = T / 1000
    P, Mo = _driver_push(pos, mom, field, T0, dt)(1000)
    u = Mo / (M_ * C)
    assert np.abs(_gamma(Mo) - u[:, 0] - 1).max() < 1e-6
    assert np.abs(u).max() > 0.3          # the wave did move the particles


@pytest.mark.parametrize("kind", ["pw", "md", "grid"])
def test_driver_equals_explicit_loop(kind):
    """oracle_push's internal t_n = t0 + n dt and r^n sampling == the explicit loop, bitwise."""
    pos, mom, field, _, fieldfn = _setup(kind)
    dt = T / 137
    a = _driver_push(pos, mom, field, T0, dt)(50)
    b = _loop_push(pos, mom, fieldfn, T0, dt)(50)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


@pytest.mark.parametrize("kind,mutation", [
    ("pw", "t_half"), ("pw", "r_next"), ("pw", "t0_ignored"),
    ("md", "t_half"), ("md", "r_next"), ("md", "t0_ignored"),
    ("grid", "r_next"),
])
def test_pins_reject_mutated_sampling(kind, mutation):
    """The pins above are discriminating: a driver that sampled the field at t_{n+1/2},
    at r^{n+1} or ignored t0 fails them (first-order drift, or an O(1) offset)."""
    good = _pin(kind, lambda pos, mom, field, fieldfn, dt: _loop_push(pos, mom, fieldfn, T0, dt))
    assert _pin_ok(kind, good), good      # the unmutated explicit loop passes
    bad = _pin(kind, lambda pos, mom, field, fieldfn, dt: _loop_push(pos, mom, fieldfn, T0, dt,
                                                                      mutation))
    assert not _pin_ok(kind, bad), bad
