"""Pins for the oracle's gather + push (U-1..U-8): conservation laws of the
gyrocentre equations (Eqs. 2-8), RK2 order, closed forms
with drifts off, invariants (mu, w for E = 0), and the survey's RHS
transcription values."""
import math

import numpy as np
import pytest

import synth
from conftest import golden_path

ATTRS = ("psi", "theta", "zeta", "rho", "w")


def _params(orc, size="T", **over):
    cfg = synth.config(size, **over)
    return cfg, orc.make_params(cfg), orc.geometry(orc.make_params(cfg))


def _energy(cfg, X, mu):
    r = np.sqrt(2 * X["psi"])
    B = 1.0 / (1.0 + r / cfg["R0"] * np.cos(X["theta"]))
    vpar = cfg["omega0"] * B * X["rho"]
    return 0.5 * vpar * vpar + mu * B


def _run(orc, p, parts, nsteps, gp):
    Xa = {k: parts[k].copy() for k in ATTRS}
    Xb = {k: parts[k].copy() for k in ATTRS}
    for _ in range(nsteps):
        orc.push(p, 1, Xa, Xb, parts["mu"], gp)
        orc.push(p, 2, Xa, Xb, parts["mu"], gp)
    return Xa


def _interior(cfg, n, seed):
    parts = synth.load_particles(cfg, n, seed=seed)
    keep = (parts["psi"] > 0.5 * 0.35 ** 2) & (parts["psi"] < 0.5 * 0.65 ** 2)
    # moderate energies only: fast particles drift into the reflecting wall
    keep &= _energy(cfg, parts, parts["mu"]) < 3.0
    return {k: v[keep] for k, v in parts.items()}


def test_rhs_transcription(orc):
    cfg, p, _ = _params(orc, "T")
    vals = dict(l.split() for l in open(golden_path("rhs_transcription.txt")) if l.strip() and not l.startswith("#"))
    r, th = 0.5, math.pi / 3
    B = orc.bfield(p, r, th)
    assert abs(B - float(vals["B"])) < 1e-12
    rho = 1.0 / (p.omega0 * B)
    assert abs(rho - float(vals["rho_par"])) < 1e-12
    d = orc.rhs(p, [0.5 * r * r, th, 0.7, rho, 0.1], 0.5, [0.01, 0.02, 0.005])
    for name, got in zip(("psidot", "thetadot", "zetadot", "rhodot", "wdot"), d):
        ref = float(vals[name])
        assert abs(got - ref) <= 1e-9 * abs(ref), name


def test_zero_field_w_and_mu_invariant(orc):
    """E = 0 => dw/dt = 0 exactly: w bitwise constant; mu never written."""
    cfg, p, g = _params(orc)
    parts = synth.load_particles(cfg, 500, seed=2)
    gp = np.zeros((p.mzetamax + 1, g.mgrid, 3))
    mu0 = parts["mu"].copy()
    Xa = _run(orc, p, parts, 5, gp)
    assert np.array_equal(Xa["w"], parts["w"])
    assert np.array_equal(parts["mu"], mu0)


def test_zero_field_energy_rk2_order(orc):
    """With phi = 0 the kinetic energy v_par^2/2 + mu B is an exact invariant of
    U-3..U-5; RK2 conserves it to O(dt^2) globally (ratio ~4 per halving)."""
    cfg, p, g = _params(orc)
    parts = _interior(cfg, 400, 4)
    gp = np.zeros((p.mzetamax + 1, g.mgrid, 3))
    E0 = _energy(cfg, parts, parts["mu"])
    errs = []
    for dt, n in ((0.4, 10), (0.2, 20), (0.1, 40)):
        pp = orc.make_params(dict(cfg, dt=dt))
        X = _run(orc, pp, parts, n, gp)
        errs.append(np.max(np.abs(_energy(cfg, X, parts["mu"]) - E0) / E0))
    r1, r2 = errs[0] / errs[1], errs[1] / errs[2]
    assert 3.4 < r1 < 4.8 and 3.4 < r2 < 4.8, errs


def test_rk2_self_convergence(orc):
    """orbit error vs dt-halved reference decreases 4.0 +- 0.4."""
    cfg, p, g = _params(orc)
    parts = _interior(cfg, 200, 6)
    gp = np.zeros((p.mzetamax + 1, g.mgrid, 3))
    sol = []
    for dt, n in ((0.2, 10), (0.1, 20), (0.05, 40)):
        sol.append(_run(orc, orc.make_params(dict(cfg, dt=dt)), parts, n, gp))
    e1 = max(np.max(np.abs(sol[0][k] - sol[1][k])) for k in ("psi", "rho"))
    e2 = max(np.max(np.abs(sol[1][k] - sol[2][k])) for k in ("psi", "rho"))
    assert 3.6 <= e1 / e2 <= 4.4, (e1, e2)


def test_static_potential_energy(orc):
    """For a static potential and mu = 0 (so phi_bar = phi), E_kin + phi is an
    exact invariant of U-3..U-5 when g_par = d phi/d zeta along b, i.e.
    d/dzeta + (1/q) d/dtheta.  Integrated with the oracle RHS and RK2."""
    cfg, p, _ = _params(orc, "T")

    def grad(X):
        r = math.sqrt(2 * X[0])
        ph, dr_, dth, dze = synth.analytic_phi(cfg, r, X[1], X[2], amp=0.05)
        q = p.q0 + p.q2 * r * r
        return ph, [dr_, dth, dze + dth / q]

    def energy(X):
        r = math.sqrt(2 * X[0])
        B = orc.bfield(p, r, X[1])
        v = p.omega0 * B * X[3]
        return 0.5 * v * v + grad(X)[0]

    def integrate(dt, n, X):
        X = np.array(X, float)
        for _ in range(n):
            Xb = X + 0.5 * dt * orc.rhs(p, X, 0.0, grad(X)[1])
            X = X + dt * orc.rhs(p, Xb, 0.0, grad(Xb)[1])
        return X

    X0 = [0.5 * 0.5 ** 2, 0.3, 0.2, 1.2 / p.omega0, 0.0]
    E0 = energy(X0)
    e = [abs(energy(integrate(dt, int(round(2.4 / dt)), X0)) - E0) for dt in (0.08, 0.04, 0.02)]
    assert e[2] < 1e-4 * abs(E0)
    assert 3.2 < e[0] / e[1] < 4.8 and 3.2 < e[1] / e[2] < 4.8, e


def test_drift_off_closed_forms(orc):
    """drifts = 0: r constant; field-line label theta - zeta/q conserved; for
    mu = 0 theta(t) obeys (theta - theta0) + (r/R0)(sin theta - sin theta0)
    = v_par t / (q R0) (integral of dtheta/dt = v_par B/(q R0))."""
    cfg, p, g = _params(orc, drifts=0)
    p = orc.make_params(dict(cfg, drifts=0, dt=0.01))
    parts = _interior(cfg, 100, 8)
    parts["mu"][:] = 0.0
    gp = np.zeros((p.mzetamax + 1, g.mgrid, 3))
    r = np.sqrt(2 * parts["psi"])
    B0 = 1.0 / (1.0 + r / cfg["R0"] * np.cos(parts["theta"]))
    vpar = cfg["omega0"] * B0 * parts["rho"]
    q = p.q0 + p.q2 * r * r
    n = 100
    Xa = {k: parts[k].copy() for k in ATTRS}
    Xb = {k: parts[k].copy() for k in ATTRS}
    th_unwrapped = parts["theta"].copy()
    ze_unwrapped = parts["zeta"].copy()
    for _ in range(n):
        th_prev, ze_prev = Xa["theta"].copy(), Xa["zeta"].copy()
        orc.push(p, 1, Xa, Xb, parts["mu"], gp)
        orc.push(p, 2, Xa, Xb, parts["mu"], gp)
        th_unwrapped += (Xa["theta"] - th_prev + math.pi) % (2 * math.pi) - math.pi
        ze_unwrapped += (Xa["zeta"] - ze_prev + math.pi) % (2 * math.pi) - math.pi
    assert np.array_equal(Xa["psi"], parts["psi"])
    alpha0 = parts["theta"] - parts["zeta"] / q
    alpha = th_unwrapped - ze_unwrapped / q
    assert np.max(np.abs(alpha - alpha0)) < 1e-12
    t = n * p.dt
    resid = (th_unwrapped - parts["theta"]) + r / cfg["R0"] * (np.sin(th_unwrapped) - np.sin(parts["theta"])) - vpar * t / (q * cfg["R0"])
    assert np.max(np.abs(resid)) < 1e-5


def test_step_global_finite_and_conservative(orc):
    """One full oracle step (S-0: two stages of charge -> poisson_smooth ->
    field -> push) on config T: finite state, mu untouched, radial range kept."""
    cfg, p, g = _params(orc, "T")
    parts = synth.load_particles(cfg, 12100, seed=1)
    nm = orc.marker_norm(p, parts)
    mu0 = parts["mu"].copy()
    out = orc.step_global(p, parts, nm)
    for k in ATTRS:
        assert np.all(np.isfinite(parts[k]))
    assert np.array_equal(parts["mu"], mu0)
    r = np.sqrt(2 * parts["psi"])
    assert r.min() >= p.a0 - 1e-15 and r.max() <= p.a1 + 1e-15
    assert np.all((parts["zeta"] >= 0) & (parts["zeta"] < 2 * math.pi))
    ch, phi, gp = out[0]
    assert np.all(np.isfinite(phi)) and np.abs(phi).max() > 0


def test_heat_flux_closed_forms(orc):
    """Diagnostic heat flux: zero field or zero weights give 0;
    a field whose theta component is the constant c everywhere (gather exact,
    U-2) gives the closed form sum w (v_par^2/2 + mu B) (-c / (r omega0 B))."""
    cfg = synth.config("T")
    p = orc.make_params(cfg)
    g = orc.geometry(p)
    parts = synth.load_particles(cfg, 3000, seed=12, w_amp=0.1)
    zero = np.zeros((p.mzetamax + 1, g.mgrid, 3))
    assert orc.heat_flux(p, parts, zero) == 0.0
    c = 0.37
    gp = zero.copy()
    gp[..., 1] = c
    gp[..., 0] = 0.2  # g_r and g_par do not enter v_E,r
    gp[..., 2] = -1.3
    r = np.sqrt(2 * parts["psi"])
    B = 1.0 / (1.0 + r / p.R0 * np.cos(parts["theta"]))
    vpar = p.omega0 * B * parts["rho"]
    want = np.sum(parts["w"] * (0.5 * vpar ** 2 + parts["mu"] * B) * (-c / (r * p.omega0 * B)))
    got = orc.heat_flux(p, parts, gp)
    assert abs(got - want) <= 1e-12 * np.sum(np.abs(parts["w"] * (0.5 * vpar ** 2 + parts["mu"] * B) * c / (r * p.omega0 * B)))
    w0 = dict(parts, w=np.zeros_like(parts["w"]))
    assert orc.heat_flux(p, w0, gp) == 0.0
