"""Pins of the CPU oracle against what the paper and the physics fix (no GPU).

Every test here checks oracle/ against something OTHER than its own formula:
exact rational rotations, closed-form orbits, exact invariants, O(dt^2)
convergence to continuous solutions, Maxwell's equations, library spherical
Bessel functions, 50-digit hand cases, brute-force sums.  Citations: PAPER.md
line numbers (L...), SURVEY.md §8(c) readings (c...).
"""
import json
import math
import os
from fractions import Fraction

import mpmath
import numpy as np
import pytest
import scipy.special

import oracle

mpmath.mp.dps = 50


def load_golden(golden_dir):
    with open(os.path.join(golden_dir, "hand_cases.json")) as f:
        return json.load(f)


# ---------------------------------------------------------------------------
# Hand cases (L175-186).  A/B via an exact rational rotation (independent of the
# cross-product form of eq. 12), C via exact arithmetic, D from 50-digit golden.
# ---------------------------------------------------------------------------

def _rotation_closed_form(p0, tz, gamma, m, dt, n_steps):
    """Exact Boris orbit in B = z with E = 0, written as a rotation.

    Eq. 11 (L155-166) is a rotation of p about B; with t = tz z the Boris
    rotation (eq. 12-13) is exactly a rotation by -theta, cos theta =
    (1-t^2)/(1+t^2), sin theta = 2t/(1+t^2) (theta = 2 atan t).  Positions from
    eq. 7: r^N = sum_{n=1..N} dt p^{n-1/2}/(gamma m).  Fractions: exact.
    """
    c = (1 - tz * tz) / (1 + tz * tz)
    s = 2 * tz / (1 + tz * tz)
    px, py = p0
    rx = ry = Fraction(0)
    out = []
    for _ in range(n_steps):
        px, py = c * px + s * py, -s * px + c * py
        rx += dt * px / (gamma * m)
        ry += dt * py / (gamma * m)
        out.append(((px, py), (rx, ry)))
    return out


def test_hand_case_A_exact_rational(golden_dir):
    g = load_golden(golden_dir)["A"]
    # p^- = (3/4, 0, 0), gamma = 5/4, t = qB dt/(2 gamma m c) = 2/5.
    exact = _rotation_closed_form((Fraction(3, 4), Fraction(0)), Fraction(2, 5), Fraction(5, 4),
                                  Fraction(1), Fraction(1), 2)
    assert exact[0][0] == (Fraction(63, 116), Fraction(-15, 29))
    assert exact[0][1] == (Fraction(63, 145), Fraction(-12, 29))
    r, p, gam = np.array(g["r0"], float), np.array(g["p0"], float), None
    for step, key in enumerate(("step1", "step2")):
        r, p, gam = oracle.boris_step(r, p, g["q"], g["m"], g["c"], g["E"], g["B"], g["dt"])
        (epx, epy), (erx, ery) = exact[step]
        np.testing.assert_allclose(p[:2], [float(epx), float(epy)], rtol=0, atol=4e-16)
        np.testing.assert_allclose(r[:2], [float(erx), float(ery)], rtol=0, atol=8e-16)
        np.testing.assert_allclose(p, g[key]["p"], rtol=0, atol=4e-16)
        np.testing.assert_allclose(r, g[key]["r"], rtol=0, atol=8e-16)
        assert gam == pytest.approx(1.25, abs=4e-16)


def test_hand_case_B_sign_of_charge(golden_dir):
    g = load_golden(golden_dir)["B"]
    r, p, gam = oracle.boris_step(g["r0"], g["p0"], g["q"], g["m"], g["c"], g["E"], g["B"], g["dt"])
    np.testing.assert_allclose(p, g["step1"]["p"], rtol=0, atol=4e-16)
    np.testing.assert_allclose(r, g["step1"]["r"], rtol=0, atol=8e-16)
    # q -> -q mirrors the rotation: y components flip sign relative to case A.
    ga = load_golden(golden_dir)["A"]
    ra, pa, _ = oracle.boris_step(ga["r0"], ga["p0"], ga["q"], ga["m"], ga["c"], ga["E"], ga["B"],
                                  ga["dt"])
    assert p[1] == -pa[1] and p[0] == pa[0]


def test_hand_case_C_pure_electric_kick(golden_dir):
    g = load_golden(golden_dir)["C"]
    r, p, gam = oracle.boris_step(g["r0"], g["p0"], g["q"], g["m"], g["c"], g["E"], g["B"], g["dt"])
    # Exact: p = qE dt = 1/2; gamma = sqrt(5)/2; x = dt p/(gamma m) = 1/sqrt(5).
    assert p[0] == 0.5 and p[1] == 0 and p[2] == 0
    assert gam == pytest.approx(math.sqrt(5) / 2, rel=2e-16)
    assert r[0] == pytest.approx(1 / math.sqrt(5), rel=4e-16)
    np.testing.assert_allclose(r, g["step1"]["r"], rtol=4e-16, atol=0)


@pytest.mark.parametrize("case", ["D_electron", "D_proton"])
def test_hand_case_D_50_digit(golden_dir, case):
    g = load_golden(golden_dir)[case]
    r, p, gam = oracle.boris_step(g["r0"], g["p0"], g["q"], g["m"], g["c"], g["E"], g["B"], g["dt"])
    np.testing.assert_allclose(p, g["step1"]["p"], rtol=4e-15, atol=1e-300)
    np.testing.assert_allclose(r, g["step1"]["r"], rtol=4e-15, atol=1e-300)
    assert gam == pytest.approx(g["step1"]["gamma"], rel=4e-16)


def test_mixed_type_table_matches_single_types(golden_dir):
    """Type table (L202-205): a mixed ensemble equals per-type runs bitwise."""
    gd = load_golden(golden_dir)
    ge, gp = gd["D_electron"], gd["D_proton"]
    n = 7
    types = np.array([0, 1, 1, 0, 1, 0, 0], np.int16)
    pos = np.zeros((n, 3))
    mom = np.zeros((n, 3))
    params = np.array(ge["E"] + ge["B"], float)
    tq, tm = [ge["q"], gp["q"]], [ge["m"], gp["m"]]
    P, M, G = oracle.push(pos, mom, types, tq, tm, 1.0, oracle.FIELD_UNIFORM, params,
                          dt=0.5, n_steps=1)
    for i in range(n):
        g = ge if types[i] == 0 else gp
        np.testing.assert_allclose(M[i], g["step1"]["p"], rtol=4e-15, atol=1e-300)
    # bitwise equal to the single-type runs
    for j in (0, 1):
        sel = types == j
        P1, M1, G1 = oracle.push(pos[sel], mom[sel], np.zeros(sel.sum(), np.int16), [tq[j]],
                                 [tm[j]], 1.0, oracle.FIELD_UNIFORM, params, dt=0.5, n_steps=1)
        assert np.array_equal(P[sel], P1) and np.array_equal(M[sel], M1) and np.array_equal(G[sel], G1)


# ---------------------------------------------------------------------------
# Half kicks (eq. 9-10): uniform E, B = 0.
# ---------------------------------------------------------------------------

def test_uniform_E_momentum_is_exact():
    """B = 0: p^{N-1/2} = p^{-1/2} + N q E dt exactly, up to rounding."""
    q, m, c, dt, N = -1.3, 0.7, 1.0, 0.01, 1000
    E = np.array([0.3, -0.2, 0.45])
    p0 = np.array([0.1, 0.2, -0.3])
    P, M, G = oracle.push([[0, 0, 0]], [p0], [0], [q], [m], c, oracle.FIELD_UNIFORM,
                          np.r_[E, 0, 0, 0], dt=dt, n_steps=N)
    np.testing.assert_allclose(M[0], p0 + N * q * E * dt, rtol=0, atol=2e-13)


def test_hyperbolic_motion_second_order():
    """Uniform E from rest: x(t) = (mc^2/qE)(sqrt(1+(qEt/mc)^2) - 1) (relativistic
    hyperbolic motion, eq. 3-5).  p^{-1/2} = 0 at t = -dt/2; Boris converges as dt^2."""
    q, m, c, Ex = 1.0, 1.0, 1.0, 1.0
    T = 2.0
    errs = []
    for N in (100, 1000):
        dt = T / N

        def x_exact(t):
            return (m * c * c / (q * Ex)) * (math.sqrt(1 + (q * Ex * (t + dt / 2) / (m * c)) ** 2) - 1)

        x0 = x_exact(0.0)
        P, M, G = oracle.push([[x0, 0, 0]], [[0, 0, 0]], [0], [q], [m], c, oracle.FIELD_UNIFORM,
                              [Ex, 0, 0, 0, 0, 0], dt=dt, n_steps=N)
        errs.append(abs(P[0, 0] - x_exact(T)) / x_exact(T))
    ratio = errs[0] / errs[1]
    assert 95 < ratio < 105, (errs, ratio)
    assert errs[1] < 1e-6


# ---------------------------------------------------------------------------
# Rotation (eq. 11-13): |p| invariant (L159-166) and the C1 Larmor orbit.
# ---------------------------------------------------------------------------

def test_p2_invariant_pure_magnetic():
    rng = np.random.default_rng(7)
    n = 1000
    mom = rng.normal(size=(n, 3)) * 3.0
    B = rng.normal(size=(n, 3)) * 2.0
    P, M, G = oracle.push(np.zeros((n, 3)), mom, np.zeros(n, np.int16), [-1.0], [1.0], 1.0,
                          oracle.FIELD_ARRAYS, E=np.zeros((n, 3)), B=B, dt=0.3, n_steps=100)
    drift = np.abs(np.linalg.norm(M, axis=1) / np.linalg.norm(mom, axis=1) - 1)
    assert drift.max() < 1e-14


def _larmor_closed_form(r0, u0, alpha, cdt_over_gamma, N):
    """u_perp rotates by alpha per step (complex z -> z e^{i alpha});
    r_perp^N = r_perp^0 + (c dt/gamma) z0 sum_{n=1..N} e^{i n alpha} (geometric sum)."""
    z0 = u0[:, 0] + 1j * u0[:, 1]
    e = np.exp(1j * alpha)
    zN = z0 * np.exp(1j * N * alpha)
    s = z0 * e * (1 - np.exp(1j * N * alpha)) / (1 - e)
    r = r0.copy()
    r[:, 0] += cdt_over_gamma * s.real
    r[:, 1] += cdt_over_gamma * s.imag
    r[:, 2] += N * cdt_over_gamma * u0[:, 2]
    u = np.stack([zN.real, zN.imag, u0[:, 2]], axis=1)
    return r, u


def test_C1_larmor_orbit_discrete_closed_form():
    """BASELINE configs[0]: 1000 e-, uniform B, |p| = mc, dt = 0.01 T_gyro, 100 steps.

    For E = 0 the Boris orbit is exactly: rotation by alpha = -2 atan(t_z) per
    step (t_z = qB dt/(2 gamma m c), eq. 13) -- SURVEY §8(c) 'C1 Larmor orbit'.
    """
    import torch
    import synth
    w = synth.config("C1")
    d = w.generate()
    q, m = w.types[0]
    c = w.light_velocity
    B = w.uniform_B[2]
    pos = torch.stack([d["x"], d["y"], d["z"]], 1).numpy()
    mom = torch.stack([d["px"], d["py"], d["pz"]], 1).numpy()
    P, M, G = oracle.push(pos, mom, np.zeros(w.n, np.int16), [q], [m], c, oracle.FIELD_UNIFORM,
                          [0, 0, 0, 0, 0, B], dt=w.dt, n_steps=w.n_steps)
    u0 = mom / (m * c)
    gamma = math.sqrt(2.0)
    tz = q * B * w.dt / (2 * gamma * m * c)
    alpha = -2 * math.atan(tz)
    # C1 constants from SURVEY §8(c): |t| = pi/100, theta = 2 atan(pi/100).
    assert abs(tz) == pytest.approx(math.pi / 100, rel=1e-13)
    assert abs(alpha) == pytest.approx(0.062811194452840266, rel=1e-13)
    r_ref, u_ref = _larmor_closed_form(pos, u0, alpha, c * w.dt / gamma, w.n_steps)
    mc, cdt = m * c, c * w.dt
    assert np.abs(M - u_ref * mc).max() / mc < 1e-13
    assert np.abs(P - r_ref).max() / cdt < 1e-11
    np.testing.assert_allclose(G, gamma, rtol=1e-14)


def test_larmor_phase_lag_and_radius():
    """O(dt^2) phase error: per-step angle 2 atan(w dt/2) vs w dt; the discrete orbit
    radius is r_L sqrt(1 + (w dt/2)^2) (1.0004933585187405)."""
    c, m, q, B = 1.0, 1.0, 1.0, 1.0
    u_perp = 1.0
    gamma = math.sqrt(1 + u_perp ** 2)
    wc = q * B / (gamma * m * c)
    T = 2 * math.pi / wc
    dt = 0.01 * T
    N = 100
    P, M, G = oracle.push([[0, 0, 0]], [[u_perp * m * c, 0, 0]], [0], [q], [m], c,
                          oracle.FIELD_UNIFORM, [0, 0, 0, 0, 0, B], dt=dt, n_steps=N)
    # phase after N steps vs the continuous N w dt = 2 pi: lag 2.0658619e-3 rad.
    ang = math.atan2(-M[0, 1], M[0, 0]) % (2 * math.pi)
    lag = 2 * math.pi - ang
    assert lag == pytest.approx(2.0658619e-3, rel=1e-6)
    # radius from three consecutive positions (circumcircle)
    pts = []
    r, p = np.zeros(3), np.array([u_perp, 0, 0])
    for _ in range(3):
        r, p, _g = oracle.boris_step(r, p, q, m, c, [0, 0, 0], [0, 0, B], dt)
        pts.append(r[:2].copy())
    a, b, cc = (np.array(x) for x in pts)
    la, lb, lc = np.linalg.norm(b - cc), np.linalg.norm(a - cc), np.linalg.norm(a - b)
    area = abs((b - a)[0] * (cc - a)[1] - (b - a)[1] * (cc - a)[0]) / 2
    R = la * lb * lc / (4 * area)
    rL = u_perp * m * c * c / (q * B)
    assert R / rL == pytest.approx(1.0004933585187405, rel=1e-9)


# ---------------------------------------------------------------------------
# Crossed fields: E x B drift, species independent (C3 shape), O(dt^2).
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("q,m", [(-1.0, 1.0), (1.0, 1.0), (1.0, 1836.15267343)])
def test_ExB_drift_second_order(q, m):
    """E = (0, 0.5B, 0), B = B z, from rest: after K lab periods T_lab = 2 pi gamma_d^3 m c/(|q|B)
    the particle is at v_d K T_lab, v_d = c E x B/B^2 = 0.5c x."""
    c, B, K = 1.0, 1.0, 5
    E = 0.5 * B
    gd = 1 / math.sqrt(1 - (E / B) ** 2)
    Tl = 2 * math.pi * gd ** 3 * m * c / (abs(q) * B)
    vd = c * E / B
    errs = []
    for M_ in (100, 1000):
        dt = Tl / M_
        P, Mo, G = oracle.push([[0, 0, 0]], [[0, 0, 0]], [0], [q], [m], c, oracle.FIELD_UNIFORM,
                               [0, E, 0, 0, 0, B], dt=dt, n_steps=K * M_)
        errs.append(abs(P[0, 0] - vd * K * Tl) / (vd * K * Tl))
    assert errs[0] == pytest.approx(8.2e-4, rel=0.05)
    assert 90 < errs[0] / errs[1] < 110


# ---------------------------------------------------------------------------
# Plane wave (north_star analytic source): exact invariants of vacuum plane-wave
# motion -- light-front gamma - u_x = 1 from rest, canonical u_y -- converge O(dt^2).
# ---------------------------------------------------------------------------

def _plane_wave_run(a0, M_, n_periods=1.0):
    c, m, q, omega = 1.0, 1.0, -1.0, 1.0
    k = omega / c
    E0 = a0 * m * c * omega / abs(q)
    params = [E0, 1, 0, 0, 0, 1, 0, omega, k, 0.0]
    T = 2 * math.pi / omega
    dt = T / M_
    r, p = np.zeros(3), np.zeros(3)
    # the invariant's value at t_{-1/2} = -dt/2, where p^{-1/2} = 0 and x = 0
    cy0 = q * E0 / (m * c * omega) * math.sin(omega * dt / 2)
    lf, cy = [], []
    for n in range(int(n_periods * M_)):
        t = n * dt
        E, B = oracle.field_plane_wave(params, r, t)
        r_old = r
        r, p, g = oracle.boris_step(r, p, q, m, c, E, B, dt)
        u = p / (m * c)
        lf.append(abs(g - u[0] - 1.0))
        # canonical momentum u_y + (q E0/(m c w)) sin(phi) at t_{n+1/2}, x^{n+1/2}
        xh = 0.5 * (r_old[0] + r[0])
        phi = k * xh - omega * (t + dt / 2)
        cy.append(abs(u[1] + q * E0 / (m * c * omega) * math.sin(phi) - cy0))
    return max(lf), max(cy)


@pytest.mark.parametrize("a0", [0.1, 1.0])
def test_plane_wave_invariants_second_order(a0):
    lf1, cy1 = _plane_wave_run(a0, 100)
    lf2, cy2 = _plane_wave_run(a0, 1000)
    assert 80 < lf1 / lf2 < 120, (lf1, lf2)
    assert 50 < cy1 / cy2 < 150, (cy1, cy2)
    if a0 == 1.0:
        assert lf1 == pytest.approx(5.5e-5, rel=0.1)


def test_plane_wave_field_definition():
    """B = khat x E, |E| = |B|, E along ehat (reading c-PW); phase = k khat.r - w t + phi0."""
    params = [2.0, 0, 0, 1, 1, 0, 0, 3.0, 5.0, 0.25]   # khat = z, ehat = x
    r = np.array([0.1, 0.2, 0.3])
    E, B = oracle.field_plane_wave(params, r, 0.7)
    phi = 5.0 * 0.3 - 3.0 * 0.7 + 0.25
    np.testing.assert_allclose(E, [2.0 * math.cos(phi), 0, 0], atol=1e-15)
    np.testing.assert_allclose(B, [0, 2.0 * math.cos(phi), 0], atol=1e-15)


# ---------------------------------------------------------------------------
# m-dipole field (eq. 14-15 in readings c9-c13)
# ---------------------------------------------------------------------------

def _md_params(xi_star=1.0, n_terms=9, A0=1.3, omega=1.7 * 1.9, k=1.7):
    return [A0, omega, k, xi_star, n_terms]


@pytest.mark.parametrize("xi_star,n_terms", [(1.0, 9), (1.5, 7)])
def test_mdipole_radial_vs_spherical_bessel(xi_star, n_terms):
    """f1 = j1, f2 = 3 j1/xi - j0, f3 = j0 - j1/xi (c11); both branches vs scipy."""
    for xi in np.r_[np.linspace(1e-6, 0.99, 17), np.linspace(xi_star - 1e-9, 12.0, 23)]:
        g1, g2, f3 = oracle.mdipole_radial(xi, xi_star, n_terms)
        j0 = scipy.special.spherical_jn(0, xi)
        j1 = scipy.special.spherical_jn(1, xi)
        tol = 1e-15 if xi_star == 1.0 else 2e-9
        assert g1 == pytest.approx(j1 / xi, rel=tol * 10, abs=tol)
        assert f3 == pytest.approx(j0 - j1 / xi, rel=tol * 10, abs=tol)
        # g2 = (3 j1/xi - j0)/xi^2 cancels catastrophically; compare with mpmath there.
        xm = mpmath.mpf(xi)
        g2_ref = (3 * (mpmath.sin(xm) / xm ** 3 - mpmath.cos(xm) / xm ** 2) - mpmath.sin(xm) / xm) / xm ** 2
        assert g2 == pytest.approx(float(g2_ref), rel=(2e-13 if xi < 1.0 else 1e-12) if xi_star == 1.0 else 5e-8,
                                   abs=1e-300)


def test_mdipole_centre_value():
    A0, w, t = 1.3, 2.0, 0.4
    E, B = oracle.field_mdipole([A0, w, 1.7, 1.0, 9], [0, 0, 0], t)
    np.testing.assert_allclose(E, 0, atol=0)
    np.testing.assert_allclose(B, [0, 0, -(4 / 3) * A0 * math.sin(w * t)], rtol=1e-15)


@pytest.mark.parametrize("point", [(0.3, -0.7, 1.1), (0.05, 0.02, -0.04), (1.9, 0.4, -2.2)])
def test_mdipole_satisfies_maxwell(point):
    """div B = 0, dB/dt = -c rot E, dE/dt = c rot B (eq. 1-2 in vacuum, L82-86) by central
    differences.  The literal text of eq. 14 fails these at O(0.1)."""
    c, k = 1.9, 1.7
    params = [1.3, k * c, k, 1.0, 9]
    x0 = np.array(point)
    t0 = 0.2
    h = 1e-4

    def F(x, t):
        return oracle.field_mdipole(params, x, t)

    def d(fn_index, comp, axis):
        ep = np.zeros(3)
        ep[axis] = h
        return (F(x0 + ep, t0)[fn_index][comp] - F(x0 - ep, t0)[fn_index][comp]) / (2 * h)

    def dt(fn_index, comp):
        return (F(x0, t0 + h)[fn_index][comp] - F(x0, t0 - h)[fn_index][comp]) / (2 * h)

    E, B = F(x0, t0)
    scale = 1.3 * k
    divB = d(1, 0, 0) + d(1, 1, 1) + d(1, 2, 2)
    rotE = [d(0, 2, 1) - d(0, 1, 2), d(0, 0, 2) - d(0, 2, 0), d(0, 1, 0) - d(0, 0, 1)]
    rotB = [d(1, 2, 1) - d(1, 1, 2), d(1, 0, 2) - d(1, 2, 0), d(1, 1, 0) - d(1, 0, 1)]
    assert abs(divB) < 1e-7 * scale
    for i in range(3):
        assert abs(dt(1, i) + c * rotE[i]) < 1e-7 * scale * c
        assert abs(dt(0, i) - c * rotB[i]) < 1e-7 * scale * c


# ---------------------------------------------------------------------------
# Kinetic energy (c17) and the driver
# ---------------------------------------------------------------------------

def test_kinetic_energy_no_cancellation():
    m, c, w = 2.0, 3.0, 1.5
    for u in (1e-6, 1e-3, 0.5, 30.0):
        mom = np.array([[u * m * c, 0, 0]])
        gamma = np.sqrt(1 + u * u)
        ke = oracle.kinetic_energy(mom, [gamma], [w], [0], [m], c)
        ref = w * (mpmath.sqrt(1 + mpmath.mpf(u) ** 2) - 1) * m * c * c
        assert ke == pytest.approx(float(ref), rel=3e-16)


def test_neumaier_sum_exact():
    assert oracle.neumaier_sum([1.0, 1e100, 1.0, -1e100]) == 2.0
    rng = np.random.default_rng(3)
    x = rng.normal(size=10000) * 10.0 ** rng.integers(-8, 8, size=10000)
    ref = mpmath.fsum([mpmath.mpf(v) for v in x])
    assert oracle.neumaier_sum(x) == pytest.approx(float(ref), rel=2e-16, abs=1e-300)


def test_type_out_of_range_rejected():
    with pytest.raises(ValueError):
        oracle.push([[0, 0, 0]], [[0, 0, 0]], [1], [1.0], [1.0], 1.0, oracle.FIELD_UNIFORM,
                    [0] * 6, dt=1.0, n_steps=1)


def test_openmp_driver_bitwise_equal_serial():
    rng = np.random.default_rng(11)
    n = 5000
    pos = rng.normal(size=(n, 3))
    mom = rng.normal(size=(n, 3))
    E = rng.normal(size=(n, 3))
    B = rng.normal(size=(n, 3))
    args = (pos, mom, np.zeros(n, np.int16), [-1.0], [1.0], 1.0, oracle.FIELD_ARRAYS)
    a = oracle.push(*args, E=E, B=B, dt=0.05, n_steps=5, n_threads=1)
    b = oracle.push(*args, E=E, B=B, dt=0.05, n_steps=5, n_threads=4)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


# ---------------------------------------------------------------------------
# Grid field gather (reading c-grid): CIC on a periodic grid.
# ---------------------------------------------------------------------------

GRID_P = [0.25, -1.0, 0.5, 0.5, 0.3, 0.7, 5, 7, 4]   # origin, spacing, (nx, ny, nz)


def _grid_nodes(fn):
    x0, y0, z0, dx, dy, dz, nx, ny, nz = GRID_P
    k, j, i = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    X, Y, Z = x0 + i * dx, y0 + j * dy, z0 + k * dz
    return np.stack([fn(X, Y, Z, c) for c in range(3)]), np.stack([fn(X, Y, Z, 3 + c)
                                                                  for c in range(3)])


def _multilinear(x, y, z, c):
    a = [0.3, -1.1, 2.0, 0.7, -0.4, 1.3][c]
    return a + 0.5 * x - 0.25 * y + 1.5 * z + 0.1 * x * y - 0.2 * y * z + 0.3 * x * z + 0.05 * x * y * z * (c + 1)


def test_grid_gather_reproduces_multilinear_fields():
    """CIC (trilinear) weights reproduce any multilinear function exactly inside the
    grid (away from the periodic seam) -- pins the weights and the node indexing
    (anisotropic grid: a swapped axis or stride fails)."""
    gE, gB = _grid_nodes(_multilinear)
    rng = np.random.default_rng(5)
    x0, y0, z0, dx, dy, dz, nx, ny, nz = GRID_P
    for _ in range(200):
        r = np.array([x0 + rng.uniform(0, (nx - 1) * dx), y0 + rng.uniform(0, (ny - 1) * dy),
                      z0 + rng.uniform(0, (nz - 1) * dz)])
        E, B = oracle.field_grid(GRID_P, gE, gB, r)
        ref = [_multilinear(r[0], r[1], r[2], c) for c in range(6)]
        np.testing.assert_allclose(np.r_[E, B], ref, rtol=1e-13, atol=1e-13)


def test_grid_gather_nodes_periodicity_partition_of_unity():
    rng = np.random.default_rng(6)
    x0, y0, z0, dx, dy, dz, nx, ny, nz = GRID_P
    gE = rng.normal(size=(3, nz, ny, nx))
    gB = rng.normal(size=(3, nz, ny, nx))
    # exactly on a node: the node's values
    i, j, k = 3, 5, 2
    E, B = oracle.field_grid(GRID_P, gE, gB, [x0 + i * dx, y0 + j * dy, z0 + k * dz])
    np.testing.assert_allclose(E, gE[:, k, j, i], rtol=1e-15, atol=1e-15)
    np.testing.assert_allclose(B, gB[:, k, j, i], rtol=1e-15, atol=1e-15)
    # periodic: shifting by a period along each axis (and negative coordinates)
    r = np.array([0.9, -0.3, 1.1])
    E0, B0 = oracle.field_grid(GRID_P, gE, gB, r)
    for shift in ([nx * dx, 0, 0], [0, -ny * dy, 0], [0, 0, 3 * nz * dz]):
        E1, B1 = oracle.field_grid(GRID_P, gE, gB, r + np.array(shift))
        np.testing.assert_allclose(E1, E0, rtol=1e-12, atol=1e-13)
        np.testing.assert_allclose(B1, B0, rtol=1e-12, atol=1e-13)
    # across the seam: between the last node and node 0 the weights interpolate linearly
    rs = np.array([x0 + (nx - 0.5) * dx, y0, z0])
    E2, _ = oracle.field_grid(GRID_P, gE, gB, rs)
    np.testing.assert_allclose(E2, 0.5 * (gE[:, 0, 0, nx - 1] + gE[:, 0, 0, 0]), rtol=1e-14)
    # partition of unity: a constant grid is gathered as that constant
    cE = np.broadcast_to(np.array([1.5, -2.0, 0.25])[:, None, None, None], (3, nz, ny, nx))
    E3, _ = oracle.field_grid(GRID_P, cE, gB, rng.normal(size=3) * 10)
    np.testing.assert_allclose(E3, [1.5, -2.0, 0.25], rtol=2e-15)


def test_grid_push_with_constant_grid_equals_uniform_push():
    """A constant grid field is the uniform field: trajectories agree to rounding."""
    x0, y0, z0, dx, dy, dz, nx, ny, nz = GRID_P
    E = np.array([0.0, 0.5, 0.1])
    Bv = np.array([0.2, 0.0, 1.0])
    gE = np.broadcast_to(E[:, None, None, None], (3, nz, ny, nx))
    gB = np.broadcast_to(Bv[:, None, None, None], (3, nz, ny, nx))
    rng = np.random.default_rng(8)
    pos = rng.normal(size=(50, 3)) * 3
    mom = rng.normal(size=(50, 3))
    args = (pos, mom, np.zeros(50, np.int16), [-1.0], [1.0], 1.0)
    P1, M1, _ = oracle.push(*args, oracle.FIELD_GRID, GRID_P, E=gE, B=gB, dt=0.1, n_steps=50)
    P2, M2, _ = oracle.push(*args, oracle.FIELD_UNIFORM, np.r_[E, Bv], dt=0.1, n_steps=50)
    np.testing.assert_allclose(M1, M2, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(P1, P2, rtol=1e-12, atol=1e-12)


# ---------------------------------------------------------------------------
# Alternative pushers (readings c-vay, c-hc): Vay (2008) and
# Higuera-Cary (2017).  The paper only cites them (L111-113, L137-140), so they are
# pinned by the physics their authors designed them for.
# ---------------------------------------------------------------------------

ALT = [oracle.PUSHER_VAY, oracle.PUSHER_HIGUERA_CARY]


@pytest.mark.parametrize("pusher", ALT)
def test_alt_pushers_equal_boris_without_magnetic_field(pusher):
    rng = np.random.default_rng(21)
    for _ in range(50):
        r0, p0, E = rng.normal(size=3), rng.normal(size=3) * 2, rng.normal(size=3)
        a = oracle.boris_step(r0, p0, -1.0, 1.0, 1.0, E, [0, 0, 0], 0.3)
        b = oracle.boris_step(r0, p0, -1.0, 1.0, 1.0, E, [0, 0, 0], 0.3, pusher=pusher)
        np.testing.assert_allclose(b[1], a[1], rtol=1e-14, atol=1e-15)
        np.testing.assert_allclose(b[0], a[0], rtol=1e-14, atol=1e-15)


@pytest.mark.parametrize("pusher", ALT)
def test_alt_pushers_keep_the_force_free_drift(pusher):
    """E perp B, |E| < |B|: a particle moving at the drift velocity v_d = c E x B/B^2
    feels no force.  Vay and Higuera-Cary keep it exactly for ANY dt (their design
    goal); Boris does not (its gamma_n is not the drift gamma) -- the test
    discriminates."""
    c, m, q = 1.0, 1.0, -1.0
    E, B = [0.0, 0.9, 0.0], [0.0, 0.0, 1.0]
    bd = 0.9
    ud = np.array([bd / math.sqrt(1 - bd * bd), 0.0, 0.0])
    dt = 2.0   # |q| B dt/(gamma m c) ~ 0.9 rad per step: far from the small-step regime
    P, M, G = oracle.push([[0, 0, 0]], [ud * m * c], [0], [q], [m], c, oracle.FIELD_UNIFORM,
                          E + B, dt=dt, n_steps=100, pusher=pusher)
    assert np.abs(M[0] / (m * c) - ud).max() < 1e-12
    np.testing.assert_allclose(P[0], [100 * dt * bd * c, 0, 0], rtol=1e-12, atol=1e-12)
    Pb, Mb, _ = oracle.push([[0, 0, 0]], [ud * m * c], [0], [q], [m], c, oracle.FIELD_UNIFORM,
                            E + B, dt=dt, n_steps=100)
    assert np.abs(Mb[0] / (m * c) - ud).max() > 1e-2


def test_higuera_cary_conserves_energy_in_pure_magnetic_field():
    rng = np.random.default_rng(22)
    n = 200
    mom = rng.normal(size=(n, 3)) * 5
    B = rng.normal(size=(n, 3)) * 3
    P, M, G = oracle.push(np.zeros((n, 3)), mom, np.zeros(n, np.int16), [1.0], [1.0], 1.0,
                          oracle.FIELD_ARRAYS, E=np.zeros((n, 3)), B=B, dt=0.7, n_steps=100,
                          pusher=oracle.PUSHER_HIGUERA_CARY)
    assert np.abs(np.linalg.norm(M, axis=1) / np.linalg.norm(mom, axis=1) - 1).max() < 1e-13


@pytest.mark.parametrize("pusher", ALT)
def test_alt_pushers_converge_second_order_to_the_same_trajectory(pusher):
    """Random fixed E, B: every pusher approximates the same ODE (eq. 3-5) to O(dt^2),
    so its distance to Boris shrinks 100x when dt shrinks 10x."""
    rng = np.random.default_rng(23)
    n = 64
    pos, mom = rng.normal(size=(n, 3)), rng.normal(size=(n, 3))
    E, B = rng.normal(size=(n, 3)) * 0.5, rng.normal(size=(n, 3))
    diffs = []
    for N in (100, 1000):
        dt = 2.0 / N
        args = (pos, mom, np.zeros(n, np.int16), [-1.0], [1.0], 1.0, oracle.FIELD_ARRAYS)
        Pa, Ma, _ = oracle.push(*args, E=E, B=B, dt=dt, n_steps=N)
        Pb, Mb, _ = oracle.push(*args, E=E, B=B, dt=dt, n_steps=N, pusher=pusher)
        diffs.append(np.abs(Pb - Pa).max())
    assert 60 < diffs[0] / diffs[1] < 160, diffs


# ---------------------------------------------------------------------------
# Current deposition (reading c-dep): direct CIC at r^{n+1/2}.
# ---------------------------------------------------------------------------

def _vel(p, m, c):
    m = np.asarray(m, dtype=float)
    g = np.sqrt(1 + np.sum(p * p, -1) / (m * c) ** 2)
    return p / (g * m)[..., None]


def test_deposit_total_current_and_weights():
    x0, y0, z0, dx, dy, dz, nx, ny, nz = GRID_P
    vol = dx * dy * dz
    rng = np.random.default_rng(31)
    n = 500
    pos = rng.normal(size=(n, 3)) * 4
    mom = rng.normal(size=(n, 3)) * 2
    w = rng.uniform(0.5, 1.5, n)
    ty = rng.integers(0, 2, n).astype(np.int16)
    tq, tm = [-1.0, 2.0], [1.0, 3.0]
    c, dt = 1.0, 0.2
    J = oracle.deposit_current(pos, mom, w, ty, tq, tm, c, dt, GRID_P)
    v = _vel(mom, np.array(tm)[ty], c)
    total = np.sum((np.array(tq)[ty] * w)[:, None] * v, 0)
    # partition of unity: the grid holds exactly the total current sum q w v
    np.testing.assert_allclose(J.reshape(3, -1).sum(1) * vol, total, rtol=1e-12, atol=1e-12)


def test_deposit_half_step_position_and_cic_shares():
    x0, y0, z0, dx, dy, dz, nx, ny, nz = GRID_P
    vol = dx * dy * dz
    c, dt, m, q = 1.0, 0.4, 1.0, -1.0
    p = np.array([[0.3, -0.2, 0.5]])
    v = _vel(p, m, c)[0]
    node = np.array([x0 + 2 * dx, y0 + 3 * dy, z0 + 1 * dz])
    # r^{n+1} chosen so that r^{n+1/2} = r^{n+1} - dt v/2 sits exactly on node (2, 3, 1)
    J = oracle.deposit_current([node + 0.5 * dt * v], p, [1.0], [0], [q], [m], c, dt, GRID_P)
    np.testing.assert_allclose(J[:, 1, 3, 2], q * v / vol, rtol=1e-12)
    assert np.count_nonzero(np.abs(J) > 1e-14 * np.abs(J).max()) == 3
    # half-step position at a cell centre: 1/8 of the current on each of the 8 nodes
    centre = node + 0.5 * np.array([dx, dy, dz])
    J = oracle.deposit_current([centre + 0.5 * dt * v], p, [1.0], [0], [q], [m], c, dt, GRID_P)
    for kk in (1, 2):
        for jj in (3, 4):
            for ii in (2, 3):
                np.testing.assert_allclose(J[:, kk, jj, ii], q * v / vol / 8, rtol=1e-12)
    # periodic images deposit identically
    J2 = oracle.deposit_current([centre + 0.5 * dt * v + [nx * dx, -2 * ny * dy, nz * dz]], p,
                                [1.0], [0], [q], [m], c, dt, GRID_P)
    np.testing.assert_allclose(J2, J, rtol=1e-12, atol=1e-15)


def test_oracle_under_address_and_undefined_behaviour_sanitizers(tmp_path):
    """the oracle's every entry point runs clean under
    -fsanitize=address,undefined (tests/oracle_sanitize_driver.c)."""
    import subprocess
    here = os.path.dirname(os.path.abspath(__file__))
    root = os.path.dirname(here)
    exe = tmp_path / "oracle_san"
    subprocess.check_call(["gcc", "-std=c11", "-O1", "-g", "-fsanitize=address,undefined",
                           "-fno-sanitize-recover=all", "-fopenmp", "-I",
                           os.path.join(root, "oracle"), os.path.join(here,
                                                                     "oracle_sanitize_driver.c"),
                           os.path.join(root, "oracle", "boris_oracle.c"), "-lm", "-o", str(exe)])
    r = subprocess.run([str(exe)], capture_output=True, text=True,
                       env=dict(os.environ, ASAN_OPTIONS="detect_leaks=1"))
    assert r.returncode == 0, r.stdout + r.stderr
    assert "runtime error" not in r.stderr and "ERROR: AddressSanitizer" not in r.stderr
