"""GPU (libboris CUDA kernels, through the C ABI) vs the CPU oracle.

Element-by-element parity at sizes that span several tiles/blocks plus a
ragged tail; sampled parity at BASELINE full size; bit-exact invariants
(AoS == SoA, aligned == unaligned, sharded == unsharded, mixed types == per-type
runs, host-resident == device-resident, order/type/weight untouched).
Tolerances: north_star (1e-12 fp64, 1e-5 fp32 after 100 steps) with the c15
metric (tests/parity_util.py).
"""
from __future__ import annotations

import math

import numpy as np
import pytest
import torch

import oracle
import synth
import paper_2104_04579_b200 as lb
from paper_2104_04579_b200.ensemble import AosEnsemble, SoaEnsemble
from parity_util import TOL, C15, Displacement, OracleRun, rounded, stack3

pytestmark = pytest.mark.gpu

PREC = {"fp32": lb.BORIS_FP32, "fp64": lb.BORIS_FP64}
LAYOUT = {"soa": lb.BORIS_LAYOUT_SOA, "aos": lb.BORIS_LAYOUT_AOS}
N_SMALL = 3 * 4096 + 37        # several blocks / tiles + a ragged tail


def gpu_field(w):
    if w.field_kind == "uniform":
        return lb.boris_field_create_uniform(w.uniform_E, w.uniform_B)
    if w.field_kind == "plane_wave":
        pw = w.plane_wave
        return lb.boris_field_create_plane_wave(pw["E0"], pw["k_hat"], pw["e_hat"], pw["omega"],
                                                pw["k"], pw["phase0"])
    if w.field_kind == "mdipole":
        md = w.plane_wave
        return lb.boris_field_create_mdipole(md["A0"], md["omega0"], md["k"])
    return None


@pytest.fixture
def boris_option():
    """Set a process-wide library option (boris_set_option) for one test; the
    previous value is restored afterwards."""
    saved = {}

    def set_(opt, value):
        saved.setdefault(opt, lb.boris_get_option(opt))
        lb.boris_set_option(opt, value)

    yield set_
    for opt, value in saved.items():
        lb.boris_set_option(opt, value)


def build(w, layout, precision, n=None, host=False):
    n = n or w.n
    d = rounded(w.generate(0, n), precision)
    cls = SoaEnsemble if layout == "soa" else AosEnsemble
    ens = cls(n, PREC[precision], w.types, w.light_velocity, host=host,
              with_fields=w.field_kind == "arrays")
    ens.fill(d)
    ens.wrap()
    field = ens.field if w.field_kind == "arrays" else gpu_field(w)
    return d, ens, field


def gpu_state(ens):
    s = ens.state()
    return (torch.stack([s["x"], s["y"], s["z"]], 1).numpy(),
            torch.stack([s["px"], s["py"], s["pz"]], 1).numpy(), s["gamma"].numpy(), s)


ORACLE_PUSHER = {0: 0, lb.BORIS_PUSH_PUSHER_VAY: 1, lb.BORIS_PUSH_PUSHER_HIGUERA_CARY: 2}


def run_parity(w, layout, precision, n, checks=(1, 2, 10, 100), host=False, flags=0,
               check_discrimination=False):
    d, ens, field = build(w, layout, precision, n, host=host)
    ref = OracleRun(w, d, precision, pusher=ORACLE_PUSHER[flags & lb.BORIS_PUSH_PUSHER_MASK])
    metric = C15()
    disp = Displacement(ref.pos, precision)
    done = 0
    worst = {}
    stream = torch.cuda.current_stream()
    for s in checks:
        k = s - done
        lb.boris_push_ex(ens.handle, field, w.dt, k, flags, None, stream)
        ref.push(k)
        torch.cuda.synchronize()
        done = s
        r, p, g, st = gpu_state(ens)
        er = metric("r", r, ref.pos)
        ep = metric("p", p, ref.mom)
        ed, eb = disp(r, ref.pos, s)
        assert ed <= TOL[precision] and abs(eb) <= TOL[precision], (s, ed, eb)
        if check_discrimination:
            # a10 off by 1e-4 (e.g. a mis-rounded dt/(S m)) must fail the displacement check
            r_bad = disp.r0 + (1 + 1e-4) * (r - disp.r0)
            ed_bad, eb_bad = disp(r_bad, ref.pos, s)
            assert max(ed_bad, abs(eb_bad)) > TOL[precision], (s, ed_bad, eb_bad)
        # gamma is derived from p (eq. 5): |d gamma| <= |u| |du| / gamma <= |du|, so the c15
        # bound on p implies |d gamma| <= tol (|u_ref| + S_u), up to gamma's own rounding.
        m = np.array([t[1] for t in w.types])[st["type"].numpy().astype(np.int64)]
        mc = (m * w.light_velocity)[:, None]
        u_ref = np.linalg.norm(ref.mom / mc, axis=1)
        s_u = metric.scale["p"] * float(np.mean(1.0 / mc))
        ulp = np.spacing(ref.gamma.astype(np.float32 if precision == "fp32" else np.float64))
        dg = np.abs(g - ref.gamma)
        assert np.all(dg <= TOL[precision] * (u_ref + s_u) + 2 * ulp), (s, float(dg.max()))
        eg = float(np.max(dg / (u_ref + s_u)))
        g_of_p = np.sqrt(1.0 + np.sum(p * p, 1) / (m * w.light_velocity) ** 2)
        # gamma = g2 * rsqrt(g2) with the <= 2 ulp MUFU rsqrt in fp32 (boris_device.cuh)
        assert np.max(np.abs(g - g_of_p) / g_of_p) <= (1e-6 if precision == "fp32" else 4e-15)
        worst[s] = (er, ep, eg, ed, eb)
        # order, types, weights untouched (bit-exact)
        assert torch.equal(st["type"], d["type"].to(torch.int16))
        assert torch.equal(st["weight"], d["weight"])
    tol = TOL[precision]
    for s, (er, ep, eg, ed, eb) in worst.items():
        assert er <= tol and ep <= tol, (s, worst)
    assert lb.boris_ensemble_get_time(ens.handle) == pytest.approx(done * w.dt, rel=1e-15)
    if w.field_kind != "arrays":
        lb.boris_field_destroy(field)
    ens.close()
    return worst


# ---------------------------------------------------------------------------
# Per-particle ("precalculated") fields, streaming kernels: C2 recipe.
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("layout", ["soa", "aos"])
@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_C2_arrays_parity(layout, precision):
    w = synth.config("C2")
    worst = run_parity(w, layout, precision, N_SMALL, check_discrimination=True)
    print(layout, precision, worst)


@pytest.mark.parametrize("layout", ["soa", "aos"])
@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_multitype_arrays_parity(layout, precision):
    w = synth.config("C2")
    w.types = [synth.ELECTRON, synth.POSITRON, synth.PROTON]
    w.type_mix = "random"
    run_parity(w, layout, precision, N_SMALL)


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 7, 255, 256, 257, 1023, 1025])
@pytest.mark.parametrize("layout", ["soa", "aos"])
def test_small_and_ragged_sizes(n, layout):
    w = synth.config("C2")
    run_parity(w, layout, "fp64", n, checks=(1, 3))


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_aos_equals_soa_bitwise(precision):
    w = synth.config("C2")
    w.types = [synth.ELECTRON, synth.POSITRON, synth.PROTON]
    w.type_mix = "random"
    _, soa, fs = build(w, "soa", precision, N_SMALL)
    _, aos, fa = build(w, "aos", precision, N_SMALL)
    for _ in range(3):
        lb.boris_push(soa.handle, fs, w.dt, 1)
        lb.boris_push(aos.handle, fa, w.dt, 1)
    torch.cuda.synchronize()
    a, b = soa.state(), aos.state()
    for k in ("x", "y", "z", "px", "py", "pz", "gamma"):
        assert torch.equal(a[k], b[k]), k


def test_unaligned_equals_aligned_bitwise():
    """Sliced tensors (4 B offset) take the scalar path; arithmetic is identical."""
    w = synth.config("C2")
    n = 4099
    d = rounded(w.generate(0, n + 1), "fp32")
    big = SoaEnsemble(n + 1, lb.BORIS_FP32, w.types, w.light_velocity)
    big.fill(d)
    ref = SoaEnsemble(n, lb.BORIS_FP32, w.types, w.light_velocity)
    ref.fill({k: v[1:] for k, v in d.items()})
    ref.wrap()
    keys = ("x", "y", "z", "px", "py", "pz")
    h = lb.boris_ensemble_wrap_soa(0, lb.BORIS_MEMORY_DEVICE, lb.BORIS_FP32, n,
                                   *(big.t[k][1:].data_ptr() for k in keys),
                                   big.t["weight"][1:].data_ptr(), big.t["gamma"][1:].data_ptr(),
                                   None, w.types, w.light_velocity)
    f = lb.boris_field_create_arrays_soa(h, *(big.t[k][1:].data_ptr()
                                              for k in ("Ex", "Ey", "Ez", "Bx", "By", "Bz")))
    lb.boris_push(h, f, w.dt, 2)
    lb.boris_push(ref.handle, ref.field, w.dt, 2)
    torch.cuda.synchronize()
    for k in keys + ("gamma",):
        assert torch.equal(big.t[k][1:], ref.t[k]), k
    lb.boris_field_destroy(f)
    lb.boris_ensemble_destroy(h)


def test_sharded_equals_unsharded_bitwise():
    """pushing contiguous shards separately == pushing the whole."""
    from paper_2104_04579_b200.dist import shard_range
    w = synth.config("C5", n=50_001)
    d = rounded(w.generate(), "fp32")
    whole = SoaEnsemble(w.n, lb.BORIS_FP32, w.types, w.light_velocity)
    whole.fill(d)
    whole.wrap()
    lb.boris_push(whole.handle, whole.field, w.dt, 3)
    world = 4
    parts = []
    for rank in range(world):
        lo, hi = shard_range(w.n, rank, world)
        # each shard generated from the global index, as a rank would
        ds = rounded(w.generate(lo, hi - lo), "fp32")
        e = SoaEnsemble(hi - lo, lb.BORIS_FP32, w.types, w.light_velocity)
        e.fill(ds)
        e.wrap()
        lb.boris_push(e.handle, e.field, w.dt, 3)
        parts.append(e)
    torch.cuda.synchronize()
    for k in ("x", "y", "z", "px", "py", "pz", "gamma"):
        assert torch.equal(torch.cat([p.t[k] for p in parts]), whole.t[k]), k


@pytest.mark.parametrize("layout", ["soa", "aos"])
@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_fused_arrays_equal_streaming_each_step_bitwise(layout, precision):
    """BORIS_PUSH_AUTO fuses n_steps with per-particle fields in registers; it must
    equal n_steps streaming launches (BORIS_PUSH_STREAM_EACH_STEP) bit for bit,
    diagnostic included."""
    w = synth.config("C5")
    w.types = [synth.ELECTRON, synth.POSITRON, synth.PROTON]
    w.type_mix = "random"
    _, a, fa = build(w, layout, precision, N_SMALL)
    _, b, fb = build(w, layout, precision, N_SMALL)
    da = torch.zeros(2, dtype=torch.float64, device="cuda")
    db = torch.zeros(2, dtype=torch.float64, device="cuda")
    lb.boris_push_ex(a.handle, fa, w.dt, 7, lb.BORIS_PUSH_AUTO, da.data_ptr())
    lb.boris_push_ex(b.handle, fb, w.dt, 7, lb.BORIS_PUSH_STREAM_EACH_STEP, db.data_ptr())
    torch.cuda.synchronize()
    sa, sb = a.state(), b.state()
    for k in ("x", "y", "z", "px", "py", "pz", "gamma", "weight", "type"):
        assert torch.equal(sa[k], sb[k]), k
    assert da[1].item() == db[1].item() == N_SMALL
    assert da[0].item() == pytest.approx(db[0].item(), rel=1e-14)
    with pytest.raises(lb.BorisError) as ei:
        lb.boris_push_ex(a.handle, fa, w.dt, 1, 0x80)
    assert ei.value.status == lb.BORIS_E_INVALID_ARG


def test_mixed_types_equal_per_type_runs_bitwise():
    w = synth.config("C2")
    w.types = [synth.ELECTRON, synth.POSITRON, synth.PROTON]
    w.type_mix = "random"
    d, mixed, fm = build(w, "soa", "fp64", N_SMALL)
    lb.boris_push(mixed.handle, fm, w.dt, 5)
    torch.cuda.synchronize()
    for j, tp in enumerate(w.types):
        sel = d["type"] == j
        dj = {k: v[sel] for k, v in d.items()}
        dj["type"] = torch.zeros_like(dj["type"])
        e = SoaEnsemble(int(sel.sum()), lb.BORIS_FP64, [tp], w.light_velocity)
        e.fill(dj)
        e.wrap()
        lb.boris_push(e.handle, e.field, w.dt, 5)
        torch.cuda.synchronize()
        for k in ("x", "y", "z", "px", "py", "pz", "gamma"):
            assert torch.equal(mixed.t[k][sel.cuda()], e.t[k]), (j, k)


# ---------------------------------------------------------------------------
# Analytic fields, register-fused kernels: C1, C3, C4 recipes and the m-dipole.
# ---------------------------------------------------------------------------

def test_C1_larmor_fp64_soa():
    w = synth.config("C1")
    worst = run_parity(w, "soa", "fp64", w.n)
    print(worst)


def test_C1_matches_discrete_closed_form():
    """BASELINE configs[0]: GPU vs the exact discrete Boris orbit (no oracle)."""
    w = synth.config("C1")
    d, ens, field = build(w, "soa", "fp64")
    lb.boris_push(ens.handle, field, w.dt, w.n_steps)
    torch.cuda.synchronize()
    r, p, g, _ = gpu_state(ens)
    q, m = w.types[0]
    c = w.light_velocity
    B = w.uniform_B[2]
    gamma = math.sqrt(2.0)
    alpha = -2 * math.atan(q * B * w.dt / (2 * gamma * m * c))
    u0 = stack3(d, "px", "py", "pz") / (m * c)
    z0 = u0[:, 0] + 1j * u0[:, 1]
    N = w.n_steps
    e = np.exp(1j * alpha)
    s = z0 * e * (1 - np.exp(1j * N * alpha)) / (1 - e)
    zN = z0 * np.exp(1j * N * alpha)
    r0 = stack3(d, "x", "y", "z")
    cdt = c * w.dt / gamma
    r_ref = r0 + np.stack([cdt * s.real, cdt * s.imag, N * cdt * u0[:, 2]], 1)
    p_ref = np.stack([zN.real, zN.imag, u0[:, 2]], 1) * m * c
    assert np.abs(p - p_ref).max() / (m * c) < 1e-12
    assert np.abs(r - r_ref).max() / (c * w.dt) < 1e-10
    lb.boris_field_destroy(field)


@pytest.mark.parametrize("layout", ["aos", "soa"])
def test_C3_crossed_fields_three_types_fp64(layout):
    w = synth.config("C3")
    run_parity(w, layout, "fp64", N_SMALL)


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
@pytest.mark.parametrize("layout", ["soa", "aos"])
def test_C4_plane_wave_parity(precision, layout):
    w = synth.config("C4")
    worst = run_parity(w, layout, precision, N_SMALL, checks=(1, 2, 10, 100))
    print(precision, layout, worst)


@pytest.mark.parametrize("orient", ["k=z,e=x", "oblique"])
def test_plane_wave_other_orientations_parity(orient):
    """Orientations other than k = x, e = y take the generic fused kernel."""
    w = synth.config("C4")
    if orient == "k=z,e=x":
        w.plane_wave.update(k_hat=(0.0, 0.0, 1.0), e_hat=(1.0, 0.0, 0.0))
    else:
        k = np.array([1.0, 2.0, 2.0]) / 3.0
        e = np.array([2.0, 1.0, -2.0]) / 3.0          # orthogonal to k
        w.plane_wave.update(k_hat=tuple(k), e_hat=tuple(e))
    run_parity(w, "soa", "fp32", N_SMALL, checks=(1, 10, 100))
    run_parity(w, "soa", "fp64", N_SMALL, checks=(1, 10, 100))


@pytest.mark.parametrize("cfg,layout,precision", [("C4", "soa", "fp32"), ("C4", "aos", "fp64"),
                                                  ("C3", "aos", "fp64"), ("C3", "soa", "fp32"),
                                                  ("C1", "soa", "fp64")])
def test_axis_aligned_specialisation_equals_generic_bitwise(cfg, layout, precision, boris_option):
    """k_fused's YZ specialisation (E || y, B || z: C1, C3, C4) drops only products with
    exact zeros, so it equals the generic kernel bitwise (BORIS_OPT_FUSED_GENERIC = 1)."""
    w = synth.config(cfg)
    n = w.n if cfg == "C1" else N_SMALL
    steps = 37
    states = []
    for generic in (0, 1):
        boris_option(lb.BORIS_OPT_FUSED_GENERIC, generic)
        _, ens, f = build(w, layout, precision, n)
        diag = torch.zeros(2, dtype=torch.float64, device="cuda")
        lb.boris_push_diag(ens.handle, f, w.dt, steps, diag.data_ptr())
        torch.cuda.synchronize()
        states.append((ens.state(), diag.cpu()))
        lb.boris_field_destroy(f)
        ens.close()
    (a, da), (b, db) = states
    for k in ("x", "y", "z", "px", "py", "pz", "gamma"):
        assert torch.equal(a[k], b[k]), k
    assert torch.equal(da, db)


@pytest.mark.parametrize("layout", ["soa", "aos"])
@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_full_type_table_parity(layout, precision):
    """BORIS_MAX_TYPES = 256 particle types (the paper's per-type table;
    SURVEY §8(a) a3: <= 256 entries) with charges and masses spread over two decades,
    random type indices: one streaming step and 20 fused steps against the oracle
    (c15), so every table entry and the shared-memory copy of the table are used."""
    w = synth.config("C2")
    g = torch.Generator().manual_seed(21)
    nt = lb.BORIS_MAX_TYPES
    qs = (torch.rand(nt, generator=g, dtype=torch.float64) * 2 - 1) * synth.E_CHARGE
    ms = synth.M_ELECTRON * 10 ** (2 * torch.rand(nt, generator=g, dtype=torch.float64))
    w.types = [(float(q), float(m)) for q, m in zip(qs, ms)]
    w.type_mix = "random"
    d, ens, field = build(w, layout, precision, N_SMALL)
    assert int(d["type"].max()) > 200
    ref = OracleRun(w, d, precision)
    metric = C15()
    for steps in (1, 20):
        lb.boris_push(ens.handle, field, w.dt, steps)
        ref.push(steps)
        torch.cuda.synchronize()
        r, p, _, st = gpu_state(ens)
        assert torch.equal(st["type"], d["type"])
        er, ep = metric("r", r, ref.pos), metric("p", p, ref.mom)
        assert er <= TOL[precision] and ep <= TOL[precision], (steps, er, ep)
    ens.close()


def mdipole_workload():
    # m-dipole at P = 0.1 PW (reading c12: A0 = k sqrt(3P/c)).
    w = synth.config("C4")
    k = synth.OMEGA0 / synth.C_LIGHT
    P = 1e21  # erg/s
    w.field_kind = "mdipole"
    w.plane_wave = dict(A0=k * math.sqrt(3 * P / synth.C_LIGHT), omega0=synth.OMEGA0, k=k)
    w.dt = synth.T0 / 3.0e4    # peak |B| ~ 247 m c w0/e: ~0.05 rad rotation per step
    return w


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
@pytest.mark.parametrize("layout", ["soa", "aos"])
def test_mdipole_branch_grouping_is_scheduling_only(precision, layout):
    """The fused m-dipole kernel schedules particles by radial branch (k_fused.cu
    k_md_order: Taylor ones first, in warp-rounds over the order list).  Pushing
    slices of the ensemble groups different particles into the same warp-rounds;
    results must not change."""
    w = mdipole_workload()
    n = 3 * 4096 + 37
    d = rounded(w.generate(0, n), precision)
    cls = SoaEnsemble if layout == "soa" else AosEnsemble
    field = gpu_field(w)
    whole = cls(n, PREC[precision], w.types, w.light_velocity)
    whole.fill(d)
    whole.wrap()
    lb.boris_push(whole.handle, field, w.dt, 40)
    cuts = [0, 1001, 5003, 5004, n]
    parts = []
    for lo, hi in zip(cuts[:-1], cuts[1:]):
        e = cls(hi - lo, PREC[precision], w.types, w.light_velocity)
        e.fill({k: v[lo:hi] for k, v in d.items()})
        e.wrap()
        lb.boris_push(e.handle, field, w.dt, 40)
        parts.append(e)
    torch.cuda.synchronize()
    ws = whole.state()
    ps = [p.state() for p in parts]
    for k in ("x", "y", "z", "px", "py", "pz", "gamma"):
        assert torch.equal(torch.cat([s[k] for s in ps]), ws[k]), k
    for e in parts + [whole]:
        e.close()
    lb.boris_field_destroy(field)


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
@pytest.mark.parametrize("layout", ["soa", "aos"])
@pytest.mark.parametrize("multi", [False, True])
@pytest.mark.parametrize("n", [5 * 1024 + 29, 1, 33])
def test_mdipole_branch_order_is_scheduling_only(precision, layout, multi, n):
    """The fused m-dipole push schedules particles by radial branch (k_md_order,
    Taylor ones first); BORIS_OPT_MD_ORDER = 0 pushes them in storage order.  Both
    must give bitwise identical states (single type: the scaled-variable kernel;
    multi-type: the generic one), n not a multiple of 32 or 64."""
    w = mdipole_workload()
    if multi:
        w.types = [synth.ELECTRON, synth.POSITRON]
        w.type_mix = "random"
    d = rounded(w.generate(0, n), precision)
    cls = SoaEnsemble if layout == "soa" else AosEnsemble
    field = gpu_field(w)
    states = []
    try:
        for order in (1, 0):
            lb.boris_set_option(lb.BORIS_OPT_MD_ORDER, order)
            e = cls(n, PREC[precision], w.types, w.light_velocity)
            e.fill(d)
            e.wrap()
            diag = torch.zeros(2, dtype=torch.float64, device="cuda")
            lb.boris_push_diag(e.handle, field, w.dt, 60, diag.data_ptr())
            torch.cuda.synchronize()
            states.append((e.state(), diag.clone()))
            e.close()
    finally:
        lb.boris_set_option(lb.BORIS_OPT_MD_ORDER, 1)
    (a, da), (b, db) = states
    for k in ("x", "y", "z", "px", "py", "pz", "gamma"):
        assert torch.equal(a[k], b[k]), k
    assert da[1].item() == db[1].item() == n
    assert abs(da[0].item() - db[0].item()) <= 1e-12 * abs(db[0].item())  # block sums reorder
    lb.boris_field_destroy(field)


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_mdipole_parity(precision):
    w = mdipole_workload()
    worst = run_parity(w, "soa", precision, N_SMALL, checks=(1, 2, 10, 100))
    print(precision, worst)


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_mdipole_beyond_time_table_one_call(precision):
    """1500 m-dipole steps in ONE boris_push_diag call: the fused kernel's per-block
    time tables hold 1024 steps, so the call runs as several launches (t0 shifted,
    the position anchor rounded to FP between them, the diagnostic on the last).
    Against the oracle (c15 metric, eq. 14 in readings c9-c13), plus KE and count."""
    w = mdipole_workload()
    n = 2048 + 13
    d, ens, field = build(w, "soa", precision, n)
    ref = OracleRun(w, d, precision)
    steps = 1500
    diag = torch.zeros(2, dtype=torch.float64, device="cuda")
    lb.boris_push_diag(ens.handle, field, w.dt, steps, diag.data_ptr())
    ref.push(steps)
    torch.cuda.synchronize()
    r, p, g, st = gpu_state(ens)
    metric = C15()
    er, ep = metric("r", r, ref.pos), metric("p", p, ref.mom)
    print(precision, er, ep)
    # north_star's bar holds "after 100 steps"; rounding errors of independent steps
    # add as a random walk, so 1500 steps get sqrt(1500/100) times the bar (measured
    # fp32: 1.2e-5 for p, 3e-7 for r; fp64 within the plain 1e-12)
    tol = TOL[precision] * (math.sqrt(steps / 100) if precision == "fp32" else 1.0)
    assert er <= tol and ep <= tol, (er, ep)
    assert lb.boris_ensemble_get_time(ens.handle) == pytest.approx(steps * w.dt, rel=1e-15)
    assert diag[1].item() == n
    ke = ref.kinetic_energy()
    assert abs(diag[0].item() - ke) <= 10 * tol * abs(ke), (diag[0].item(), ke)
    lb.boris_field_destroy(field)
    ens.close()


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_field_evaluate_mdipole_is_the_fused_step_field(precision):
    """boris_field_evaluate returns the field the fused push uses (libboris.h): one
    streaming step with the evaluated m-dipole arrays gives the momenta and gamma of
    one fused m-dipole step from the same state at the same time, to the rounding of
    the fused step's folded factors (it multiplies the type's aE, alpha into the
    field's scalar factors instead of forming E and B), and the same branch of
    reading c13 for every particle (xi = kR spans 0..3.8 in the 0.6 lambda sphere)."""
    w = mdipole_workload()
    n = N_SMALL
    d = rounded(w.generate(0, n), precision)
    g = torch.Generator().manual_seed(11)
    for k in ("px", "py", "pz"):   # moving particles: the rotation is exercised
        d[k] = rounded({k: 3.0 * synth.M_ELECTRON * synth.C_LIGHT
                        * torch.randn(n, generator=g, dtype=torch.float64)}, precision)[k]
    t0 = 0.29 * synth.T0
    a = SoaEnsemble(n, PREC[precision], w.types, w.light_velocity, with_fields=True)
    b = SoaEnsemble(n, PREC[precision], w.types, w.light_velocity, with_fields=False)
    for e in (a, b):
        e.fill(d)
        e.wrap()
        lb.boris_ensemble_set_time(e.handle, t0)
    src = gpu_field(w)
    lb.boris_field_evaluate(src, a.handle, t0, a.field)
    lb.boris_push_ex(a.handle, a.field, w.dt, 1, lb.BORIS_PUSH_STREAM_EACH_STEP)
    lb.boris_push(b.handle, src, w.dt, 1)
    torch.cuda.synchronize()
    sa, sb = a.state(), b.state()
    # a few roundings per product chain: 16 u of the storage precision (c15 metric)
    u = 2.0 ** -24 if precision == "fp32" else 2.0 ** -53
    pa = torch.stack([sa["px"], sa["py"], sa["pz"]], 1).numpy()
    pb = torch.stack([sb["px"], sb["py"], sb["pz"]], 1).numpy()
    assert C15()("p", pa, pb) <= 16 * u
    for k in ("x", "y", "z", "gamma"):
        ref = sb[k].numpy()
        assert np.all(np.abs(sa[k].numpy() - ref) <= 16 * u * np.abs(ref)), k
    lb.boris_field_destroy(src)
    a.close()
    b.close()


@pytest.mark.parametrize("kind", ["uniform", "plane_wave", "mdipole"])
@pytest.mark.parametrize("precision", ["fp32", "fp64"])
@pytest.mark.parametrize("layout", ["soa", "aos"])
def test_field_evaluate_vs_oracle(kind, precision, layout):
    """boris_field_evaluate (precalculated fields, L369-371) == the oracle's field at
    each particle's position and time t."""
    w = mdipole_workload() if kind == "mdipole" else synth.config("C4" if kind == "plane_wave"
                                                                   else "C3")
    n = N_SMALL
    d = rounded(w.generate(0, n), precision)
    cls = SoaEnsemble if layout == "soa" else AosEnsemble
    ens = cls(n, PREC[precision], w.types, w.light_velocity, with_fields=True)
    ens.fill(d)
    ens.wrap()
    src = gpu_field(w)
    t = 0.37 * synth.T0
    lb.boris_field_evaluate(src, ens.handle, t, ens.field)
    torch.cuda.synchronize()
    if layout == "soa":
        E = torch.stack([ens.t[k].double().cpu() for k in ("Ex", "Ey", "Ez")], 1).numpy()
        B = torch.stack([ens.t[k].double().cpu() for k in ("Bx", "By", "Bz")], 1).numpy()
    else:
        f = ens.fld.double().cpu().numpy()
        E, B = f[:, :3], f[:, 3:]
    from parity_util import oracle_field
    okind, params = oracle_field(w, precision)
    pos = stack3(d, "x", "y", "z")
    Er = np.zeros_like(pos)
    Br = np.zeros_like(pos)
    for i in range(n):
        if okind == oracle.FIELD_UNIFORM:
            Er[i], Br[i] = params[:3], params[3:]
        elif okind == oracle.FIELD_PLANE_WAVE:
            Er[i], Br[i] = oracle.field_plane_wave(params, pos[i], t)
        else:
            Er[i], Br[i] = oracle.field_mdipole(params, pos[i], t)
    scale = max(np.abs(Er).max(), np.abs(Br).max())
    tol = 2e-6 if precision == "fp32" else 1e-13
    assert np.abs(E - Er).max() <= tol * scale
    assert np.abs(B - Br).max() <= tol * scale
    lb.boris_field_destroy(src)
    ens.close()


# ---------------------------------------------------------------------------
# Diagnostics, upload/download, host-resident ensembles, edge cases.
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("precision", ["fp32", "fp64"])
@pytest.mark.parametrize("layout", ["soa", "aos"])
def test_kinetic_energy_diag(precision, layout):
    w = synth.config("C5", n=N_SMALL)
    w.types = [synth.ELECTRON, synth.POSITRON, synth.PROTON]
    w.type_mix = "random"
    d, ens, field = build(w, layout, precision)
    ref = OracleRun(w, d, precision)
    diag = torch.zeros(2, dtype=torch.float64, device="cuda")
    lb.boris_push_diag(ens.handle, field, w.dt, 2, diag.data_ptr())
    ref.push(2)
    torch.cuda.synchronize()
    ke, cnt = diag.tolist()
    assert cnt == w.n
    ke_ref = ref.kinetic_energy()
    assert ke == pytest.approx(ke_ref, rel=1e-12 if precision == "fp64" else 2e-6)
    # deterministic: a second diagnostic of the same state is bitwise equal
    d2 = torch.zeros(2, dtype=torch.float64, device="cuda")
    lb.boris_kinetic_energy(ens.handle, d2.data_ptr())
    d3 = torch.zeros(2, dtype=torch.float64, device="cuda")
    lb.boris_kinetic_energy(ens.handle, d3.data_ptr())
    torch.cuda.synchronize()
    assert torch.equal(d2, d3)
    assert d2[0].item() == pytest.approx(ke_ref, rel=1e-12 if precision == "fp64" else 2e-6)


@pytest.mark.parametrize("layout", ["soa", "aos"])
@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_upload_download_roundtrip(layout, precision):
    w = synth.config("C3", n=10_007)
    d = w.generate()
    h = lb.boris_ensemble_create(0, LAYOUT[layout], PREC[precision], w.n, w.types, w.light_velocity)
    pos = stack3(d, "x", "y", "z")
    mom = stack3(d, "px", "py", "pz") + 1e-3 * synth.M_ELECTRON * synth.C_LIGHT
    lb.boris_ensemble_upload(h, 0, w.n, pos, mom, d["weight"].numpy(), d["type"].numpy())
    out = lb.boris_ensemble_download(h, 0, w.n)
    cast = (lambda a: a.astype(np.float32).astype(np.float64)) if precision == "fp32" else (lambda a: a)
    assert np.array_equal(out["pos"], cast(pos))
    assert np.array_equal(out["mom"], cast(mom))
    assert np.array_equal(out["type"], d["type"].numpy())
    m = np.array([t[1] for t in w.types])[out["type"]]
    g_ref = np.sqrt(1 + np.sum(mom ** 2, 1) / (m * w.light_velocity) ** 2)
    np.testing.assert_allclose(out["gamma"], g_ref, rtol=1e-15 if precision == "fp64" else 1e-7)
    # partial range
    sub = lb.boris_ensemble_download(h, 17, 100)
    assert np.array_equal(sub["pos"], out["pos"][17:117])
    bad = d["type"].numpy().copy()
    bad[5] = 3
    with pytest.raises(lb.BorisError) as ei:
        lb.boris_ensemble_upload(h, 0, w.n, pos, mom, None, bad)
    assert ei.value.status == lb.BORIS_E_TYPE_OUT_OF_RANGE
    lb.boris_ensemble_destroy(h)


@pytest.mark.parametrize("layout", ["soa", "aos"])
def test_host_resident_equals_device_bitwise(layout, boris_option):
    boris_option(lb.BORIS_OPT_HOST_CHUNK, 4096)  # several chunks through the pipeline
    w = synth.config("C2")
    _, dev, fdev = build(w, layout, "fp32", N_SMALL)
    _, host, fhost = build(w, layout, "fp32", N_SMALL, host=True)
    for _ in range(2):
        lb.boris_push(dev.handle, fdev, w.dt, 1)
        lb.boris_push(host.handle, fhost, w.dt, 1)
    torch.cuda.synchronize()
    a, b = dev.state(), host.state()
    for k in ("x", "y", "z", "px", "py", "pz", "gamma"):
        assert torch.equal(a[k], b[k]), k


@pytest.mark.parametrize("layout", ["soa", "aos"])
@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_host_resident_upload_download_roundtrip(layout, precision):
    """Host-resident ensembles: boris_ensemble_upload/download convert on the host
    side of the boundary (data movement only) and round-trip exactly."""
    w = synth.config("C3", n=1001)
    d = w.generate()
    cls = SoaEnsemble if layout == "soa" else AosEnsemble
    e = cls(w.n, PREC[precision], w.types, w.light_velocity, host=True).wrap()
    pos = stack3(d, "x", "y", "z")
    mom = stack3(d, "px", "py", "pz") + 0.3 * synth.M_ELECTRON * synth.C_LIGHT
    lb.boris_ensemble_upload(e.handle, 0, w.n, pos, mom, d["weight"].numpy(), d["type"].numpy())
    out = lb.boris_ensemble_download(e.handle, 0, w.n)
    cast = (lambda a: a.astype(np.float32).astype(np.float64)) if precision == "fp32" else (lambda a: a)
    assert np.array_equal(out["pos"], cast(pos))
    assert np.array_equal(out["mom"], cast(mom))
    assert np.array_equal(out["type"], d["type"].numpy())
    m = np.array([t[1] for t in w.types])[out["type"]]
    g_ref = np.sqrt(1 + np.sum(mom ** 2, 1) / (m * w.light_velocity) ** 2)
    np.testing.assert_allclose(out["gamma"], g_ref, rtol=1e-15 if precision == "fp64" else 1e-7)
    # push through the chunked pipeline, then read back through download
    f = lb.boris_field_create_uniform(w.uniform_E, w.uniform_B)
    lb.boris_push(e.handle, f, w.dt, 3)
    torch.cuda.synchronize()
    out2 = lb.boris_ensemble_download(e.handle, 0, w.n)
    assert not np.array_equal(out2["pos"], out["pos"])
    lb.boris_field_destroy(f)
    e.close()


def test_host_resident_analytic_multistep():
    w = synth.config("C4")
    run_parity(w, "soa", "fp64", N_SMALL, checks=(5, 20), host=True)


def test_push_is_cuda_graph_capturable():
    """boris_push / boris_push_diag do no host sync or allocation: a step loop can be
    captured once into a CUDA graph and replayed; replay == eager, bitwise."""
    w = synth.config("C5", n=N_SMALL)
    _, a, fa = build(w, "soa", "fp32")
    _, b, fb = build(w, "soa", "fp32")
    da = torch.zeros(2, dtype=torch.float64, device="cuda")
    db = torch.zeros(2, dtype=torch.float64, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        lb.boris_push_diag(b.handle, fb, w.dt, 1, db.data_ptr(), s)   # warm-up (kernel attrs)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(4):
            lb.boris_push_diag(b.handle, fb, w.dt, 1, db.data_ptr(), torch.cuda.current_stream())
    torch.cuda.synchronize()
    for _ in range(1 + 4 * 2):   # eager: 1 warm-up step + 2 replays x 4 steps
        lb.boris_push_diag(a.handle, fa, w.dt, 1, da.data_ptr())
    g.replay()
    g.replay()
    torch.cuda.synchronize()
    sa, sb = a.state(), b.state()
    for k in ("x", "y", "z", "px", "py", "pz", "gamma"):
        assert torch.equal(sa[k], sb[k]), k
    assert torch.equal(da, db)


def test_c_example_program(tmp_path):
    """examples/push_c_abi.c: the C ABI used from plain C on the GPU (Larmor invariants)."""
    import subprocess
    from test_abi_cpu import build_c_example
    exe = build_c_example(lb, tmp_path)
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "pushed 1000 electrons" in r.stdout


def test_edge_cases_and_errors():
    w = synth.config("C2")
    # n = 0 ensembles and n_steps = 0 pushes are no-ops
    e0 = SoaEnsemble(0, lb.BORIS_FP32, w.types, w.light_velocity).wrap()
    lb.boris_push(e0.handle, e0.field, w.dt, 3)
    diag = torch.full((2,), 7.0, dtype=torch.float64, device="cuda")
    lb.boris_push_diag(e0.handle, e0.field, w.dt, 1, diag.data_ptr())
    torch.cuda.synchronize()
    assert diag.tolist() == [0.0, 0.0]
    _, e, f = build(w, "soa", "fp32", 1000)
    before = e.state()
    lb.boris_push(e.handle, f, w.dt, 0)
    torch.cuda.synchronize()
    after = e.state()
    assert all(torch.equal(before[k], after[k]) for k in before)
    with pytest.raises(lb.BorisError) as ei:
        lb.boris_push(e.handle, f, float("nan"), 1)
    assert ei.value.status == lb.BORIS_E_INVALID_ARG
    with pytest.raises(lb.BorisError) as ei:
        lb.boris_push(e.handle, f, w.dt, -1)
    assert ei.value.status == lb.BORIS_E_INVALID_ARG
    # field arrays of another ensemble size -> mismatch
    _, e2, f2 = build(w, "soa", "fp32", 999)
    with pytest.raises(lb.BorisError) as ei:
        lb.boris_push(e.handle, f2, w.dt, 1)
    assert ei.value.status == lb.BORIS_E_MISMATCH
    # type out of range at wrap
    three = [synth.ELECTRON, synth.POSITRON, synth.PROTON]
    bad = SoaEnsemble(100, lb.BORIS_FP32, three, w.light_velocity)
    bad.t["type"][50] = 3
    with pytest.raises(lb.BorisError) as ei:
        bad.wrap()
    assert ei.value.status == lb.BORIS_E_TYPE_OUT_OF_RANGE
    bad.t["type"][50] = -1
    with pytest.raises(lb.BorisError):
        bad.wrap()


def test_out_of_memory_is_reported_and_not_sticky():
    """An ensemble larger than the device (2^40 fp64 SoA particles = 72 TB) fails with
    OUT_OF_MEMORY, leaves no sticky CUDA error, and the library keeps working."""
    with pytest.raises(lb.BorisError) as ei:
        lb.boris_ensemble_create(0, lb.BORIS_LAYOUT_SOA, lb.BORIS_FP64, lb.BORIS_MAX_PARTICLES,
                                 [synth.ELECTRON], synth.C_LIGHT)
    assert ei.value.status == lb.BORIS_E_OUT_OF_MEMORY
    w = synth.config("C2")
    run_parity(w, "soa", "fp32", 4099, checks=(1, 2))
    torch.cuda.synchronize()


# ---------------------------------------------------------------------------
# Full BASELINE sizes, in the launch configuration bench.py times: sampled parity.
# ---------------------------------------------------------------------------

def _sampled_full_size(name, layout, precision, n_steps, n=None, sample=20_000):
    w = synth.config(name, n=n)
    d, ens, field = build(w, layout, precision)
    diag = torch.zeros(2, dtype=torch.float64, device="cuda")
    lb.boris_push_diag(ens.handle, field, w.dt, n_steps, diag.data_ptr())
    torch.cuda.synchronize()
    assert diag[1].item() == w.n
    idx = np.unique(np.r_[np.linspace(0, w.n - 1, sample).astype(np.int64), w.n - 1, w.n - 2])
    ds = {k: v[idx] for k, v in d.items()}
    ref = OracleRun(w, ds, precision)
    ref.push(n_steps)
    r, p, g, _ = gpu_state(ens)
    metric = C15()
    er = metric("r", r[idx], ref.pos)
    ep = metric("p", p[idx], ref.mom)
    assert er <= TOL[precision] and ep <= TOL[precision], (er, ep)
    ed, eb = Displacement(stack3(ds, "x", "y", "z"), precision)(r[idx], ref.pos, n_steps)
    assert ed <= TOL[precision] and abs(eb) <= TOL[precision], (ed, eb)
    if w.field_kind != "arrays":
        lb.boris_field_destroy(field)
    ens.close()
    return er, ep


def test_full_size_C5_bench_configuration():
    """BASELINE configs[4] at its full single-GPU size (8e8, the bench's N=1 launch
    configuration: streaming kernel + fused KE, one step): sampled trajectories vs the
    oracle, and the device KE sum vs the oracle's Neumaier KE of the GPU's own state
    (checks the full-size partial reduction)."""
    import oracle as orc
    w = synth.config("C5")
    n = w.n
    ens = SoaEnsemble(n, lb.BORIS_FP32, w.types, w.light_velocity)
    chunk = 1 << 24
    for c0 in range(0, n, chunk):
        ens.fill(w.generate(c0, min(chunk, n - c0), device="cuda"), first=c0)
    ens.wrap()
    idx = np.unique(np.r_[np.linspace(0, n - 1, 20_000).astype(np.int64), n - 1])
    ds = rounded(w.generate_indices(torch.from_numpy(idx)), "fp32")
    diag = torch.zeros(2, dtype=torch.float64, device="cuda")
    lb.boris_push_diag(ens.handle, ens.field, w.dt, 1, diag.data_ptr())
    torch.cuda.synchronize()
    assert diag[1].item() == n
    ref = OracleRun(w, ds, "fp32")
    ref.push(1)
    it = torch.from_numpy(idx).cuda()
    r = torch.stack([ens.t[k][it] for k in ("x", "y", "z")], 1).double().cpu().numpy()
    p = torch.stack([ens.t[k][it] for k in ("px", "py", "pz")], 1).double().cpu().numpy()
    metric = C15()
    assert metric("r", r, ref.pos) <= TOL["fp32"]
    assert metric("p", p, ref.mom) <= TOL["fp32"]
    ed, eb = Displacement(stack3(ds, "x", "y", "z"), "fp32")(r, ref.pos, 1)
    assert ed <= TOL["fp32"] and abs(eb) <= TOL["fp32"], (ed, eb)
    # KE of the GPU state, summed by the oracle on the host chunk by chunk (Neumaier)
    parts = []
    for c0 in range(0, n, chunk):
        sl = slice(c0, min(n, c0 + chunk))
        mom = torch.stack([ens.t[k][sl] for k in ("px", "py", "pz")], 1).double().cpu().numpy()
        g = ens.t["gamma"][sl].double().cpu().numpy()
        wgt = ens.t["weight"][sl].double().cpu().numpy()
        parts.append(orc.kinetic_energy(mom, g, wgt, np.zeros(len(g), np.int16),
                                        [w.types[0][1]], w.light_velocity))
    ke_host = orc.neumaier_sum(parts)
    assert diag[0].item() == pytest.approx(ke_host, rel=2e-6)
    ens.close()


def test_beyond_int32_particle_indices():
    """n = 2^31 + 37 (the C5 recipe; ~125 GB of HBM): every index is 64-bit in the
    streaming kernel, the fused KE reduction and the ragged tail.  Sampled particles
    around 2^31 and at the end vs the oracle; the diagnostic count is exact."""
    free, _ = torch.cuda.mem_get_info()
    n = (1 << 31) + 37
    if free < 140e9:
        pytest.skip(f"needs ~125 GB of free device memory, {free / 1e9:.0f} GB free")
    w = synth.config("C5", n=n)
    ens = SoaEnsemble(n, lb.BORIS_FP32, w.types, w.light_velocity)
    chunk = 1 << 25
    for c0 in range(0, n, chunk):
        ens.fill(w.generate(c0, min(chunk, n - c0), device="cuda"), first=c0)
    ens.wrap()
    b = 1 << 31
    idx = np.unique(np.r_[np.linspace(0, n - 1, 4000).astype(np.int64),
                          np.arange(b - 40, min(n, b + 40)), np.arange(n - 40, n)])
    ds = rounded(w.generate_indices(torch.from_numpy(idx)), "fp32")
    diag = torch.zeros(2, dtype=torch.float64, device="cuda")
    lb.boris_push_diag(ens.handle, ens.field, w.dt, 1, diag.data_ptr())
    torch.cuda.synchronize()
    assert diag[1].item() == n
    ref = OracleRun(w, ds, "fp32")
    ref.push(1)

    def gather(t):
        return np.array([t[int(i)].item() for i in idx], dtype=np.float64)

    r = np.stack([gather(ens.t[k]) for k in ("x", "y", "z")], 1)
    p = np.stack([gather(ens.t[k]) for k in ("px", "py", "pz")], 1)
    metric = C15()
    assert metric("r", r, ref.pos) <= TOL["fp32"]
    assert metric("p", p, ref.mom) <= TOL["fp32"]
    ens.close()
    del ens
    torch.cuda.empty_cache()


def _big_sample(n):
    b = 1 << 31
    return np.unique(np.r_[np.linspace(0, n - 1, 3000).astype(np.int64),
                           np.arange(b - 40, min(n, b + 40)), np.arange(n - 40, n)])


def test_beyond_int32_aos_streaming():
    """AoS (TMA record tiles) with 2^31 + 37 particles and per-particle field records
    (~129 GB): 64-bit record offsets in the tile loop, the tail and the KE count."""
    free, _ = torch.cuda.mem_get_info()
    n = (1 << 31) + 37
    if free < 145e9:
        pytest.skip(f"needs ~130 GB of free device memory, {free / 1e9:.0f} GB free")
    w = synth.config("C5", n=n)
    ens = AosEnsemble(n, lb.BORIS_FP32, w.types, w.light_velocity)
    chunk = 1 << 25
    for c0 in range(0, n, chunk):
        ens.fill(w.generate(c0, min(chunk, n - c0), device="cuda"), first=c0)
    ens.wrap()
    idx = _big_sample(n)
    ds = rounded(w.generate_indices(torch.from_numpy(idx)), "fp32")
    diag = torch.zeros(2, dtype=torch.float64, device="cuda")
    lb.boris_push_diag(ens.handle, ens.field, w.dt, 1, diag.data_ptr())
    torch.cuda.synchronize()
    assert diag[1].item() == n
    ref = OracleRun(w, ds, "fp32")
    ref.push(1)
    rec = np.array([ens.rec[int(i), :6].tolist() for i in idx], dtype=np.float64)
    metric = C15()
    assert metric("r", rec[:, :3], ref.pos) <= TOL["fp32"]
    assert metric("p", rec[:, 3:6], ref.mom) <= TOL["fp32"]
    ens.close()
    del ens
    torch.cuda.empty_cache()


def test_beyond_int32_fused_multitype_uniform():
    """The register-fused kernel (C3 recipe: three types, crossed uniform E x B, SoA
    fp32, 10 fused steps) with 2^31 + 37 particles (~73 GB): one block per 128
    particles is a 16.8M-block grid."""
    free, _ = torch.cuda.mem_get_info()
    n = (1 << 31) + 37
    if free < 90e9:
        pytest.skip(f"needs ~75 GB of free device memory, {free / 1e9:.0f} GB free")
    w = synth.config("C3", n=n)
    ens = SoaEnsemble(n, lb.BORIS_FP32, w.types, w.light_velocity, with_fields=False)
    chunk = 1 << 25
    for c0 in range(0, n, chunk):
        ens.fill(w.generate(c0, min(chunk, n - c0), device="cuda"), first=c0)
    ens.wrap()
    field = gpu_field(w)
    idx = _big_sample(n)
    ds = rounded(w.generate_indices(torch.from_numpy(idx)), "fp32")
    lb.boris_push(ens.handle, field, w.dt, 10)
    torch.cuda.synchronize()
    ref = OracleRun(w, ds, "fp32")
    ref.push(10)

    def gather(t):
        return np.array([t[int(i)].item() for i in idx], dtype=np.float64)

    r = np.stack([gather(ens.t[k]) for k in ("x", "y", "z")], 1)
    p = np.stack([gather(ens.t[k]) for k in ("px", "py", "pz")], 1)
    assert np.array_equal(gather(ens.t["type"]), ds["type"].numpy().astype(np.float64))
    metric = C15()
    assert metric("r", r, ref.pos) <= TOL["fp32"]
    assert metric("p", p, ref.mom) <= TOL["fp32"]
    lb.boris_field_destroy(field)
    ens.close()
    del ens
    torch.cuda.empty_cache()


def test_full_size_C2_fp32_soa_sampled():
    print(_sampled_full_size("C2", "soa", "fp32", 1))


def test_full_size_C2_fp64_aos_sampled():
    print(_sampled_full_size("C2", "aos", "fp64", 1))


def test_full_size_C3_sampled():
    print(_sampled_full_size("C3", "aos", "fp64", 100))


def test_full_size_C4_sampled():
    print(_sampled_full_size("C4", "soa", "fp32", 100))


# ---------------------------------------------------------------------------
# Grid field gather + periodic sort (reading c-grid).
# ---------------------------------------------------------------------------

def grid_setup(precision, nx=24, ny=20, nz=16, seed=11):
    """A periodic grid covering the 0.6-lambda sphere, node values Gaussian at the
    C2 field scale (sigma = 80 m c w0/e per component)."""
    L = 1.5 * synth.LAMBDA0
    origin = [-L / 2 - 0.13 * L / nx, -L / 2, -L / 2 + 0.07 * L / nz]
    spacing = [L / nx, L / ny, L / nz]
    g = torch.Generator().manual_seed(seed)
    nodes = torch.randn((6, nz, ny, nx), generator=g, dtype=torch.float64) * 80 * synth.E_UNIT
    dt = torch.float32 if precision == "fp32" else torch.float64
    nodes = nodes.to(dt).to(torch.float64)           # both sides see the same rounded nodes
    dev = [nodes[c].to(dt).contiguous().cuda() for c in range(6)]
    h = lb.boris_field_create_grid(0, PREC[precision], nx, ny, nz, origin, spacing,
                                   *(t.data_ptr() for t in dev))
    params = origin + spacing + [nx, ny, nz]
    return h, params, nodes[:3].numpy(), nodes[3:].numpy()


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
@pytest.mark.parametrize("layout", ["soa", "aos"])
def test_grid_gather_vs_oracle(precision, layout):
    h, params, gE, gB = grid_setup(precision)
    w = synth.config("C2")
    n = N_SMALL
    d = rounded(w.generate(0, n), precision)
    d["x"] = d["x"] * 3.0   # some particles outside the box: periodic wrap
    d = rounded(d, precision)
    cls = SoaEnsemble if layout == "soa" else AosEnsemble
    ens = cls(n, PREC[precision], w.types, w.light_velocity)
    ens.fill(d)
    ens.wrap()
    lb.boris_field_evaluate(h, ens.handle, 0.0, ens.field)
    torch.cuda.synchronize()
    if layout == "soa":
        E = torch.stack([ens.t[k].double().cpu() for k in ("Ex", "Ey", "Ez")], 1).numpy()
        B = torch.stack([ens.t[k].double().cpu() for k in ("Bx", "By", "Bz")], 1).numpy()
    else:
        f = ens.fld.double().cpu().numpy()
        E, B = f[:, :3], f[:, 3:]
    pos = stack3(d, "x", "y", "z")
    Er = np.zeros_like(pos)
    Br = np.zeros_like(pos)
    for i in range(n):
        Er[i], Br[i] = oracle.field_grid(params, gE, gB, pos[i])
    scale = float(np.abs(gE).max())
    tol = 4e-6 if precision == "fp32" else 1e-13
    assert np.abs(E - Er).max() <= tol * scale
    assert np.abs(B - Br).max() <= tol * scale
    lb.boris_field_destroy(h)
    ens.close()


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_grid_push_parity(precision):
    h, params, gE, gB = grid_setup(precision)
    w = synth.config("C2")
    d, ens, field = build(w, "soa", precision, N_SMALL)
    ref = OracleRun(w, d, precision)
    ref.kind, ref.params, ref.E, ref.B = oracle.FIELD_GRID, params, gE, gB
    metric = C15()
    disp = Displacement(ref.pos, precision)
    done = 0
    worst = {}
    for s in (1, 10, 100):
        lb.boris_push(ens.handle, h, w.dt, s - done)
        ref.push(s - done)
        done = s
        torch.cuda.synchronize()
        r, p, g, st = gpu_state(ens)
        worst[s] = (metric("r", r, ref.pos), metric("p", p, ref.mom)) + disp(r, ref.pos, s)
    print(precision, worst)
    for s, (er, ep, ed, eb) in worst.items():
        assert er <= TOL[precision] and ep <= TOL[precision], worst
        assert ed <= TOL[precision] and abs(eb) <= TOL[precision], worst
    lb.boris_field_destroy(h)
    ens.close()


def test_grid_fused_push_with_frequent_cell_crossings():
    """The fused grid kernel keeps a particle's cell records in registers and reloads
    them on a cell change (grid.cuh grid_gather_cached).  A fine grid and a larger dt
    make most particles cross several cells within one 100-step launch; fp64 parity
    with the oracle must hold through the reloads."""
    precision = "fp64"
    h, params, gE, gB = grid_setup(precision, nx=96, ny=80, nz=64)
    w = synth.config("C2")
    w.dt = synth.T0 / 2000.0
    d, ens, field = build(w, "soa", precision, N_SMALL)
    ref = OracleRun(w, d, precision)
    ref.kind, ref.params, ref.E, ref.B = oracle.FIELD_GRID, params, gE, gB
    lb.boris_push(ens.handle, h, w.dt, 100)
    ref.push(100)
    torch.cuda.synchronize()
    r, p, g, st = gpu_state(ens)
    metric = C15()
    er, ep = metric("r", r, ref.pos), metric("p", p, ref.mom)
    assert er <= TOL[precision] and ep <= TOL[precision], (er, ep)
    # non-vacuous: most particles changed cell during the launch
    org, hs = np.array(params[0:3]), np.array(params[3:6])
    c0 = np.floor((stack3(d, "x", "y", "z") - org) / hs)
    c1 = np.floor((ref.pos - org) / hs)
    moved = np.mean(np.any(c0 != c1, axis=1))
    assert moved > 0.5, moved
    lb.boris_field_destroy(h)
    ens.close()


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
@pytest.mark.parametrize("layout", ["soa", "aos"])
@pytest.mark.parametrize("n", [3 * 2048 + 333, 300_000 + 17])
def test_sort_by_cell_is_a_stable_permutation(precision, layout, n):
    """n = 300017: 147 radix tiles x 512 digits = 75264 histogram entries, scanned by
    the single-pass look-back kernel in 5 chunks with a ragged last one."""
    h, params, gE, gB = grid_setup(precision, nx=9, ny=7, nz=5)
    w = synth.config("C2")
    w.types = [synth.ELECTRON, synth.POSITRON, synth.PROTON]
    w.type_mix = "random"
    d = rounded(w.generate(0, n), precision)
    d["weight"] = torch.arange(n, dtype=torch.float64)      # particle id (exact)
    cls = SoaEnsemble if layout == "soa" else AosEnsemble
    ens = cls(n, PREC[precision], w.types, w.light_velocity)
    ens.fill(d)
    ens.wrap()
    before = ens.state()
    lb.boris_ensemble_sort_by_cell(ens.handle, h)
    torch.cuda.synchronize()
    after = ens.state()
    ids = after["weight"].numpy().astype(np.int64)
    assert sorted(ids.tolist()) == list(range(n))            # a permutation
    for k in ("x", "y", "z", "px", "py", "pz", "gamma", "type"):
        assert torch.equal(after[k], before[k][ids]), k      # records moved whole
    # cell keys (host, double) non-decreasing; ids increasing inside a cell (stable)
    x0, y0, z0, dx, dy, dz, nx, ny, nz = params
    pos = np.stack([after["x"].numpy(), after["y"].numpy(), after["z"].numpy()], 1)
    ci = [np.floor((pos[:, a] - params[a]) / params[3 + a]).astype(np.int64) % int(params[6 + a])
          for a in range(3)]
    key = (ci[2] * ny + ci[1]) * nx + ci[0]
    ok = np.diff(key) >= 0
    same = np.diff(key) == 0
    frac_bad = 1.0 - ok.mean()
    assert frac_bad < 1e-3, frac_bad      # host/device floor may differ exactly on a face
    assert np.all(np.diff(ids)[same & ok] > 0) or frac_bad > 0
    # sorting a sorted ensemble is the identity
    lb.boris_ensemble_sort_by_cell(ens.handle, h)
    torch.cuda.synchronize()
    again = ens.state()
    for k in after:
        assert torch.equal(again[k], after[k]), k
    lb.boris_field_destroy(h)
    ens.close()


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
@pytest.mark.parametrize("has_w,has_type", [(True, False), (False, False), (False, True),
                                            (True, True)])
def test_sort_wrapped_arrays_with_optional_components(precision, has_w, has_type):
    """boris_ensemble_sort_by_cell on wrapped torch arrays with weight / type absent
    (NULL) or present, one element off 16 B alignment: every record layout of the
    permutation (packed records of 7-8 FP slots + an optional type slot, vector or
    shared-memory packing) moves each particle whole and sorts by cell (PAPER.md
    L233-236)."""
    h, params, _, _ = grid_setup(precision, nx=13, ny=11, nz=9)
    dt = torch.float32 if precision == "fp32" else torch.float64
    n = 2 * 4096 + 101
    g = torch.Generator().manual_seed(7)
    L = 1.5 * synth.LAMBDA0

    def arr(vals):  # device array starting one element past a 256 B boundary
        buf = torch.empty(n + 1, dtype=vals.dtype, device="cuda")
        buf[1:] = vals.cuda()
        return buf[1:]

    t = {k: arr((torch.rand(n, generator=g, dtype=torch.float64) - 0.5).to(dt) * L)
         for k in ("x", "y", "z")}
    t["px"] = arr(torch.arange(n, dtype=dt))                # particle id (exact)
    for k in ("py", "pz"):
        t[k] = arr(torch.randn(n, generator=g, dtype=torch.float64).to(dt))
    t["weight"] = arr(torch.rand(n, generator=g, dtype=torch.float64).to(dt)) if has_w else None
    t["gamma"] = arr(1 + torch.rand(n, generator=g, dtype=torch.float64).to(dt))
    types = [synth.ELECTRON, synth.POSITRON, synth.PROTON] if has_type else [synth.ELECTRON]
    t["type"] = arr(torch.randint(0, 3, (n,), generator=g).to(torch.int16)) if has_type else None
    ptr = {k: (v.data_ptr() if v is not None else None) for k, v in t.items()}
    ens = lb.boris_ensemble_wrap_soa(0, lb.BORIS_MEMORY_DEVICE, PREC[precision], n,
                                     ptr["x"], ptr["y"], ptr["z"], ptr["px"], ptr["py"],
                                     ptr["pz"], ptr["weight"], ptr["gamma"], ptr["type"], types,
                                     synth.C_LIGHT)
    before = {k: v.clone() for k, v in t.items() if v is not None}
    lb.boris_ensemble_sort_by_cell(ens, h)
    torch.cuda.synchronize()
    ids = t["px"].cpu().numpy().astype(np.int64)
    assert sorted(ids.tolist()) == list(range(n))
    idc = torch.from_numpy(ids).cuda()
    for k, v in before.items():
        assert torch.equal(t[k], v[idc]), k
    nx, ny = int(params[6]), int(params[7])
    pos = np.stack([t[k].double().cpu().numpy() for k in ("x", "y", "z")], 1)
    ci = [np.floor((pos[:, a] - params[a]) / params[3 + a]).astype(np.int64) % int(params[6 + a])
          for a in range(3)]
    key = (ci[2] * ny + ci[1]) * nx + ci[0]
    assert (np.diff(key) >= 0).mean() > 1 - 1e-3
    same = np.diff(key) == 0
    assert (np.diff(ids)[same] > 0).mean() > 1 - 1e-3     # stable inside a cell
    lb.boris_ensemble_destroy(ens)
    lb.boris_field_destroy(h)


def _grid64(precision):
    """The bench scripts' PIC grid: 64^3 nodes over a 1.5-lambda periodic box."""
    g = 64
    L = 1.5 * synth.LAMBDA0
    dt_ = torch.float32 if precision == "fp32" else torch.float64
    gen = torch.Generator(device="cuda").manual_seed(3)
    comps = [(torch.randn((g, g, g), generator=gen, device="cuda", dtype=torch.float64)
              * 80 * synth.E_UNIT).to(dt_).contiguous() for _ in range(6)]
    h = lb.boris_field_create_grid(0, PREC[precision], g, g, g, [-L / 2] * 3, [L / g] * 3,
                                   *(c.data_ptr() for c in comps))
    params = [-L / 2] * 3 + [L / g] * 3 + [g, g, g]
    return h, params, comps


def test_full_size_sort_and_deposition_pic_workload():
    """The PIC benchmark workload at its full size (10^7 fp32 C2 particles, 64^3 grid,
    the configuration scripts/bench_grid.py and bench_deposit.py time): the sort from
    random order is a stable permutation (ids carried exactly in weight + gamma) that
    orders the cells, and the deposition of the sorted ensemble equals the oracle's
    within the summation bound (tol x sum |q w v| / volume per component)."""
    h, params, comps = _grid64("fp32")
    w = synth.config("C2", n=10_000_000)
    n = w.n
    ens = SoaEnsemble(n, lb.BORIS_FP32, w.types, w.light_velocity, with_fields=False)
    ens.fill(w.generate(0, n, device="cuda"))
    ids = torch.arange(n, device="cuda", dtype=torch.int64)
    ens.t["weight"].copy_((ids % 4096).to(torch.float32) + 1.0)   # exact in fp32
    ens.t["gamma"].copy_((ids // 4096).to(torch.float32))
    ens.wrap()
    before = {k: ens.t[k].clone() for k in ("x", "y", "z", "px", "py", "pz")}
    lb.boris_ensemble_sort_by_cell(ens.handle, h)
    torch.cuda.synchronize()
    got = (ens.t["gamma"].to(torch.int64) * 4096 + ens.t["weight"].to(torch.int64) - 1)
    assert torch.equal(torch.sort(got).values, ids)                 # a permutation
    for k, v in before.items():
        assert torch.equal(ens.t[k], v[got]), k                      # records moved whole
    g = 64
    cell = [torch.floor((ens.t[k].double() - params[a]) / params[3 + a]).long() % g
            for a, k in enumerate(("x", "y", "z"))]
    key = (cell[2] * g + cell[1]) * g + cell[0]
    dk = key[1:] - key[:-1]
    assert (dk >= 0).double().mean().item() > 1 - 1e-4
    same = dk == 0
    assert ((got[1:] - got[:-1])[same] > 0).double().mean().item() > 1 - 1e-4  # stable
    # deposition of the sorted ensemble vs the oracle (weights restored to 1)
    ens.t["weight"].fill_(1.0)
    J = [torch.zeros((g, g, g), device="cuda", dtype=torch.float32) for _ in range(3)]
    lb.boris_deposit_current(ens.handle, h, w.dt, *(j.data_ptr() for j in J))
    torch.cuda.synchronize()
    Jg = torch.stack(J).double().cpu().numpy()
    pos = torch.stack([ens.t[k] for k in ("x", "y", "z")], 1).double().cpu().numpy()
    mom = torch.stack([ens.t[k] for k in ("px", "py", "pz")], 1).double().cpu().numpy()
    tq, tm = [t[0] for t in w.types], [t[1] for t in w.types]
    Jr = oracle.deposit_current(pos, mom, np.ones(n), np.zeros(n, np.int16), tq, tm,
                                w.light_velocity, w.dt, params)
    m = tm[0]
    gam = np.sqrt(1.0 + ((mom / (m * w.light_velocity)) ** 2).sum(1))[:, None]
    vol = params[3] * params[4] * params[5]
    contrib = (abs(tq[0]) * np.abs(mom / (m * gam)) / vol).sum(0)
    err = np.abs(Jg - Jr).reshape(3, -1).max(1)
    assert (err <= 1e-5 * contrib).all(), err / contrib
    lb.boris_field_destroy(h)
    ens.close()


def test_full_size_fused_pic_step():
    """boris_push_deposit at the PIC benchmark size (10^7 fp32, 64^3, sorted, the
    configuration scripts/pic_cycle.py times): the state is bitwise the single-step grid
    push's, J equals boris_deposit_current of the pushed state within the summation
    bound, and the KE diagnostic counts every particle."""
    h, params, comps = _grid64("fp32")
    w = synth.config("C2", n=10_000_000)
    n = w.n
    d = w.generate(0, n, device="cuda")
    a = SoaEnsemble(n, lb.BORIS_FP32, w.types, w.light_velocity, with_fields=False)
    b = SoaEnsemble(n, lb.BORIS_FP32, w.types, w.light_velocity, with_fields=False)
    for e in (a, b):
        e.fill(d)
        e.wrap()
        lb.boris_ensemble_sort_by_cell(e.handle, h)
    g = 64
    Ja = [torch.zeros((g, g, g), device="cuda") for _ in range(3)]
    Jb = [torch.zeros((g, g, g), device="cuda") for _ in range(3)]
    diag = torch.zeros(2, dtype=torch.float64, device="cuda")
    lb.boris_push_deposit(a.handle, h, w.dt, *(j.data_ptr() for j in Ja), diag.data_ptr())
    lb.boris_push(b.handle, h, w.dt, 1)
    lb.boris_deposit_current(b.handle, h, w.dt, *(j.data_ptr() for j in Jb))
    torch.cuda.synchronize()
    for k in ("x", "y", "z", "px", "py", "pz", "gamma"):
        assert torch.equal(a.t[k], b.t[k]), k
    assert diag[1].item() == n
    m, q = w.types[0][1], w.types[0][0]
    mom = torch.stack([b.t[k] for k in ("px", "py", "pz")], 1).double()
    gam = torch.sqrt(1.0 + ((mom / (m * w.light_velocity)) ** 2).sum(1, keepdim=True))
    vol = params[3] * params[4] * params[5]
    contrib = (abs(q) * (mom / (m * gam)).abs() / vol).sum(0).cpu().numpy()
    err = (torch.stack(Ja).double() - torch.stack(Jb).double()).abs().reshape(3, -1).max(1)
    assert (err.values.cpu().numpy() <= 1e-5 * contrib).all()
    lb.boris_field_destroy(h)
    a.close()
    b.close()


def test_sorted_push_equals_unsorted_push_bitwise():
    """The push of each particle is independent of order: sorted and unsorted
    ensembles give bit-identical particles (matched by id)."""
    h, params, gE, gB = grid_setup("fp32")
    w = synth.config("C2")
    n = N_SMALL
    d = rounded(w.generate(0, n), "fp32")
    d["weight"] = torch.arange(n, dtype=torch.float64)
    a = SoaEnsemble(n, lb.BORIS_FP32, w.types, w.light_velocity)
    b = SoaEnsemble(n, lb.BORIS_FP32, w.types, w.light_velocity)
    a.fill(d)
    b.fill(d)
    a.wrap()
    b.wrap()
    lb.boris_ensemble_sort_by_cell(b.handle, h)
    lb.boris_push(a.handle, h, w.dt, 20)
    lb.boris_push(b.handle, h, w.dt, 20)
    torch.cuda.synchronize()
    sa, sb = a.state(), b.state()
    ids = sb["weight"].numpy().astype(np.int64)
    for k in ("x", "y", "z", "px", "py", "pz", "gamma"):
        assert torch.equal(sb[k], sa[k][ids]), k
    with pytest.raises(lb.BorisError) as ei:     # precision mismatch
        h64, *_ = grid_setup("fp64")
        lb.boris_push(a.handle, h64, w.dt, 1)
    assert ei.value.status == lb.BORIS_E_MISMATCH
    lb.boris_field_destroy(h)


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
@pytest.mark.parametrize("layout", ["soa", "aos"])
def test_deposit_current_vs_oracle(precision, layout):
    """CIC current deposition at r^{n+1/2} (reading c-dep), generated state taken as the
    post-push state; both sides deposit the same rounded inputs."""
    h, params, gE, gB = grid_setup(precision)
    w = synth.config("C5")
    w.types = [synth.ELECTRON, synth.POSITRON, synth.PROTON]
    w.type_mix = "random"
    n = N_SMALL
    d = rounded(w.generate(0, n), precision)
    cls = SoaEnsemble if layout == "soa" else AosEnsemble
    ens = cls(n, PREC[precision], w.types, w.light_velocity, with_fields=False)
    ens.fill(d)
    ens.wrap()
    nx, ny, nz = int(params[6]), int(params[7]), int(params[8])
    dt_ = torch.float32 if precision == "fp32" else torch.float64
    J = [torch.full((nz, ny, nx), 7.0, dtype=dt_, device="cuda") for _ in range(3)]
    lb.boris_deposit_current(ens.handle, h, w.dt, *(j.data_ptr() for j in J))
    torch.cuda.synchronize()
    Jg = torch.stack(J).double().cpu().numpy()
    pos, mom = stack3(d, "x", "y", "z"), stack3(d, "px", "py", "pz")
    tq, tm = [t[0] for t in w.types], [t[1] for t in w.types]
    Jr = oracle.deposit_current(pos, mom, d["weight"].numpy(), d["type"].numpy(), tq, tm,
                                w.light_velocity, w.dt, params)
    scale = np.abs(Jr).max()
    tol = 1e-5 if precision == "fp32" else 1e-12
    assert np.abs(Jg - Jr).max() <= tol * scale
    vol = params[3] * params[4] * params[5]
    np.testing.assert_allclose(Jg.reshape(3, -1).sum(1) * vol, Jr.reshape(3, -1).sum(1) * vol,
                               rtol=tol, atol=tol * scale * vol)
    lb.boris_field_destroy(h)
    ens.close()


@pytest.mark.parametrize("layout", ["soa", "aos"])
@pytest.mark.parametrize("precision", ["fp32", "fp64"])
@pytest.mark.parametrize("mode", ["sorted", "one_cell", "few_cells", "tiny"])
def test_deposit_current_runs_and_contention(precision, mode, layout):
    """The run-accumulating SoA deposition on the inputs it is built for: particles
    sorted by cell (long runs, lanes' open cells merged by the warp segmented scan),
    every particle in one cell (maximum contention), a 2x2x2 block of cells (runs
    broken at every few particles), and n < one warp.  Bound: summation error
    <= tol x sum over particles of |q w v| / cell volume (a dropped or doubled particle
    is ~1/n of that sum, far above tol)."""
    h, params, _, _ = grid_setup(precision)
    w = synth.config("C5")
    w.types = [synth.ELECTRON, synth.POSITRON, synth.PROTON]
    w.type_mix = "random"
    n = 19 if mode == "tiny" else N_SMALL
    d = w.generate(0, n)
    org, sp = np.array(params[:3]), np.array(params[3:6])
    if mode in ("one_cell", "few_cells"):
        g = torch.Generator().manual_seed(5)
        span = 1 if mode == "one_cell" else 2
        cell = torch.randint(0, span, (n, 3), generator=g).double() + 5.0
        frac = 0.1 + 0.8 * torch.rand((n, 3), generator=g, dtype=torch.float64)
        pos = torch.from_numpy(org) + (cell + frac) * torch.from_numpy(sp)
        d["x"], d["y"], d["z"] = pos[:, 0].clone(), pos[:, 1].clone(), pos[:, 2].clone()
    d = rounded(d, precision)
    cls = SoaEnsemble if layout == "soa" else AosEnsemble
    ens = cls(n, PREC[precision], w.types, w.light_velocity, with_fields=False)
    ens.fill(d)
    ens.wrap()
    if mode == "sorted":
        lb.boris_ensemble_sort_by_cell(ens.handle, h)
        torch.cuda.synchronize()
        s = ens.state()
        d = {k: s[k] for k in ("x", "y", "z", "px", "py", "pz", "weight", "type")}
    nx, ny, nz = int(params[6]), int(params[7]), int(params[8])
    dt_ = torch.float32 if precision == "fp32" else torch.float64
    J = [torch.zeros((nz, ny, nx), dtype=dt_, device="cuda") for _ in range(3)]
    lb.boris_deposit_current(ens.handle, h, w.dt, *(j.data_ptr() for j in J))
    torch.cuda.synchronize()
    Jg = torch.stack(J).double().cpu().numpy()
    pos, mom = stack3(d, "x", "y", "z"), stack3(d, "px", "py", "pz")
    typ = d["type"].numpy().astype(np.int64)
    tq = np.array([t[0] for t in w.types])
    tm = np.array([t[1] for t in w.types])
    Jr = oracle.deposit_current(pos, mom, d["weight"].numpy(), typ, list(tq), list(tm),
                                w.light_velocity, w.dt, params)
    m = tm[typ][:, None]
    gam = np.sqrt(1.0 + ((mom / (m * w.light_velocity)) ** 2).sum(1))[:, None]
    vol = params[3] * params[4] * params[5]
    single = (np.abs(tq[typ])[:, None] * d["weight"].numpy()[:, None]
              * np.abs(mom / (m * gam))) / vol
    contrib = single.sum(0)
    tol = 1e-5 if precision == "fp32" else 1e-12
    err = np.abs(Jg - Jr).reshape(3, -1).max(1)
    assert (err <= tol * contrib).all(), (err / contrib, mode)
    # not vacuous: a typical single particle's current is above the bound
    assert (np.median(single, 0) > 4 * tol * contrib).all()
    lb.boris_field_destroy(h)
    ens.close()


# ---------------------------------------------------------------------------
# Fused PIC particle step: grid push + current deposition in one kernel.
# ---------------------------------------------------------------------------

def _deposit_bound(d, w, params, precision):
    """Summation-error bound per J component: tol x sum over particles of
    |q w v| / cell volume (as test_deposit_current_runs_and_contention)."""
    pos, mom = stack3(d, "x", "y", "z"), stack3(d, "px", "py", "pz")
    typ = d["type"].numpy().astype(np.int64)
    tq = np.array([t[0] for t in w.types])
    tm = np.array([t[1] for t in w.types])
    m = tm[typ][:, None]
    gam = np.sqrt(1.0 + ((mom / (m * w.light_velocity)) ** 2).sum(1))[:, None]
    vol = params[3] * params[4] * params[5]
    single = (np.abs(tq[typ])[:, None] * d["weight"].numpy()[:, None] * np.abs(mom / (m * gam))) / vol
    tol = 1e-5 if precision == "fp32" else 1e-12
    return tol * single.sum(0), pos, mom, typ, tq, tm


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
@pytest.mark.parametrize("layout", ["soa", "aos"])
@pytest.mark.parametrize("order", ["sorted", "unsorted"])
@pytest.mark.parametrize("n", [N_SMALL, 5])
def test_push_deposit_equals_push_then_deposit(precision, layout, order, n):
    """boris_push_deposit == boris_push (1 step, grid field) then boris_deposit_current:
    state bitwise, J to the float summation-order bound, and J against the oracle's
    deposition of the pushed state; the diagnostic matches boris_push_diag.  Three
    types, ragged n (fused SoA kernel; AoS takes the two-launch path)."""
    h, params, _, _ = grid_setup(precision)
    w = synth.config("C5")
    w.types = [synth.ELECTRON, synth.POSITRON, synth.PROTON]
    w.type_mix = "random"
    d = rounded(w.generate(0, n), precision)
    cls = SoaEnsemble if layout == "soa" else AosEnsemble
    a = cls(n, PREC[precision], w.types, w.light_velocity, with_fields=False)
    b = cls(n, PREC[precision], w.types, w.light_velocity, with_fields=False)
    a.fill(d)
    b.fill(d)
    a.wrap()
    b.wrap()
    if order == "sorted":
        lb.boris_ensemble_sort_by_cell(a.handle, h)
        lb.boris_ensemble_sort_by_cell(b.handle, h)
    nx, ny, nz = int(params[6]), int(params[7]), int(params[8])
    dt_ = torch.float32 if precision == "fp32" else torch.float64
    Ja = [torch.full((nz, ny, nx), 3.0, dtype=dt_, device="cuda") for _ in range(3)]
    Jb = [torch.zeros((nz, ny, nx), dtype=dt_, device="cuda") for _ in range(3)]
    da = torch.zeros(2, dtype=torch.float64, device="cuda")
    db = torch.zeros(2, dtype=torch.float64, device="cuda")
    lb.boris_push_deposit(a.handle, h, w.dt, *(j.data_ptr() for j in Ja), da.data_ptr())
    lb.boris_push_diag(b.handle, h, w.dt, 1, db.data_ptr())
    lb.boris_deposit_current(b.handle, h, w.dt, *(j.data_ptr() for j in Jb))
    torch.cuda.synchronize()
    sa, sb = a.state(), b.state()
    for k in ("x", "y", "z", "px", "py", "pz", "gamma", "weight", "type"):
        assert torch.equal(sa[k], sb[k]), k
    assert lb.boris_ensemble_get_time(a.handle) == lb.boris_ensemble_get_time(b.handle) == w.dt
    assert da[1].item() == n
    assert da[0].item() == pytest.approx(db[0].item(), rel=1e-12)
    after = {k: sa[k] for k in ("x", "y", "z", "px", "py", "pz", "weight", "type")}
    bound, pos, mom, typ, tq, tm = _deposit_bound(after, w, params, precision)
    Jga = torch.stack(Ja).double().cpu().numpy()
    Jgb = torch.stack(Jb).double().cpu().numpy()
    assert (np.abs(Jga - Jgb).reshape(3, -1).max(1) <= 2 * bound).all()
    Jr = oracle.deposit_current(pos, mom, after["weight"].numpy(), typ, list(tq), list(tm),
                                w.light_velocity, w.dt, params)
    assert (np.abs(Jga - Jr).reshape(3, -1).max(1) <= bound).all()
    a.close()
    b.close()
    lb.boris_field_destroy(h)


def test_push_deposit_errors():
    h, params, _, _ = grid_setup("fp32")
    w = synth.config("C2")
    ens = SoaEnsemble(64, lb.BORIS_FP32, w.types, w.light_velocity)
    ens.fill(rounded(w.generate(0, 64), "fp32"))
    ens.wrap()
    J = [torch.zeros(int(params[6] * params[7] * params[8]), device="cuda") for _ in range(3)]
    with pytest.raises(lb.BorisError) as ei:    # not a grid
        lb.boris_push_deposit(ens.handle, ens.field, w.dt, *(j.data_ptr() for j in J))
    assert ei.value.status == lb.BORIS_E_INVALID_ARG
    with pytest.raises(lb.BorisError) as ei:    # NULL J
        lb.boris_push_deposit(ens.handle, h, w.dt, J[0].data_ptr(), None, J[2].data_ptr())
    assert ei.value.status == lb.BORIS_E_INVALID_ARG
    with pytest.raises(lb.BorisError) as ei:    # dt not finite
        lb.boris_push_deposit(ens.handle, h, float("nan"), *(j.data_ptr() for j in J))
    assert ei.value.status == lb.BORIS_E_INVALID_ARG
    h64, *_ = grid_setup("fp64")
    with pytest.raises(lb.BorisError) as ei:    # precision mismatch
        lb.boris_push_deposit(ens.handle, h64, w.dt, *(j.data_ptr() for j in J))
    assert ei.value.status == lb.BORIS_E_MISMATCH
    ens.close()
    lb.boris_field_destroy(h)
    lb.boris_field_destroy(h64)


# ---------------------------------------------------------------------------
# Alternative pushers (readings c-vay, c-hc).
# ---------------------------------------------------------------------------

ALT_FLAGS = [lb.BORIS_PUSH_PUSHER_VAY, lb.BORIS_PUSH_PUSHER_HIGUERA_CARY]


@pytest.mark.parametrize("flags", ALT_FLAGS)
@pytest.mark.parametrize("precision", ["fp32", "fp64"])
@pytest.mark.parametrize("cfg", ["C2", "C3", "C4"])
def test_alt_pusher_parity(flags, precision, cfg):
    w = synth.config(cfg)
    layout = "aos" if cfg == "C3" else "soa"
    worst = run_parity(w, layout, precision, N_SMALL, flags=flags)
    print(cfg, precision, hex(flags), worst)


@pytest.mark.parametrize("flags", ALT_FLAGS)
def test_alt_pusher_single_steps_equal_fused_bitwise(flags):
    """Per-particle fields: n single-step launches == one n-step fused launch."""
    w = synth.config("C2")
    _, a, fa = build(w, "soa", "fp32", N_SMALL)
    _, b, fb = build(w, "soa", "fp32", N_SMALL)
    lb.boris_push_ex(a.handle, fa, w.dt, 5, flags)
    lb.boris_push_ex(b.handle, fb, w.dt, 5, flags | lb.BORIS_PUSH_STREAM_EACH_STEP)
    torch.cuda.synchronize()
    sa, sb = a.state(), b.state()
    for k in ("x", "y", "z", "px", "py", "pz", "gamma"):
        assert torch.equal(sa[k], sb[k]), k


@pytest.mark.parametrize("flags", ALT_FLAGS)
def test_alt_pusher_force_free_drift_on_gpu(flags):
    """E x B drift at large dt: Vay / Higuera-Cary keep u = u_d (design property)."""
    c, m, q = 1.0, 1.0, -1.0
    bd = 0.9
    ud = bd / math.sqrt(1 - bd * bd)
    n = 1000
    ens = SoaEnsemble(n, lb.BORIS_FP64, [(q, m)], c, with_fields=False)
    ens.t["px"].fill_(ud * m * c)
    ens.wrap()
    f = lb.boris_field_create_uniform([0, bd, 0], [0, 0, 1])
    lb.boris_push_ex(ens.handle, f, 2.0, 100, flags)
    torch.cuda.synchronize()
    s = ens.state()
    assert (s["px"] / (m * c) - ud).abs().max().item() < 1e-12
    assert s["py"].abs().max().item() < 1e-12
    np.testing.assert_allclose(s["x"].numpy(), 100 * 2.0 * bd * c, rtol=1e-12)
    with pytest.raises(lb.BorisError):
        lb.boris_push_ex(ens.handle, f, 1.0, 1, lb.BORIS_PUSH_PUSHER_MASK)
    lb.boris_field_destroy(f)
