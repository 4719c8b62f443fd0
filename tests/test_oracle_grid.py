"""Pins for the oracle's LIGHT grid kernels (F-1..F-5): smooth, zonal solve,
gyro operator, weighted Jacobi, field gradients."""
import math

import numpy as np
import pytest

import synth

TWO_PI = 2 * math.pi


@pytest.fixture(scope="module")
def T(orc):
    cfg = synth.config("T")
    p = orc.make_params(cfg)
    return cfg, p, orc.geometry(p)


def _node_coords(p, g):
    """Per node of planes 0..K: ring r, physical theta, plane zeta."""
    K = p.mzetamax
    r = np.zeros((K + 1, g.mgrid))
    th = np.zeros((K + 1, g.mgrid))
    ze = np.zeros((K + 1, g.mgrid))
    for k in range(K + 1):
        for i in range(p.mpsi + 1):
            j = np.arange(g.mtheta[i] + 1)
            sl = slice(g.igrid[i], g.igrid[i] + g.mtheta[i] + 1)
            r[k, sl] = p.a0 + i * (p.a1 - p.a0) / p.mpsi
            th[k, sl] = j * TWO_PI / g.mtheta[i] + k * TWO_PI / K * g.qtinv[i]
            ze[k, sl] = k * TWO_PI / K
    return r, th, ze


def test_smooth_preserves_constants(orc, T):
    cfg, p, g = T
    f = np.full((p.mzetamax + 1, g.mgrid), 2.5)
    assert np.max(np.abs(orc.smooth(p, f) - 2.5)) < 1e-14


def test_smooth_is_linear(orc, T):
    cfg, p, g = T
    rng = np.random.default_rng(0)
    a = rng.standard_normal((p.mzetamax + 1, g.mgrid))
    b = rng.standard_normal((p.mzetamax + 1, g.mgrid))
    lhs = orc.smooth(p, 2 * a - 3 * b)
    rhs = 2 * orc.smooth(p, a) - 3 * orc.smooth(p, b)
    assert np.max(np.abs(lhs - rhs)) < 1e-13


def test_zonal_solve_quadratic_exact(orc):
    """phi00 = (r - a0)(a1 - r) solves -rho^2 (1/r)(r phi')' = rho^2 (4r - a0 - a1)/r;
    the second-order scheme is exact for quadratics."""
    cfg = synth.config("A")
    p = orc.make_params(cfg)
    r = p.a0 + np.arange(p.mpsi + 1) * (p.a1 - p.a0) / p.mpsi
    rho2 = 1.0 / p.omega0 ** 2
    nbar = rho2 * (4 * r - p.a0 - p.a1) / r
    phi00 = orc.zonal_solve(p, nbar)
    assert np.max(np.abs(phi00 - (r - p.a0) * (p.a1 - r))) < 1e-11


def test_gyro_op_constant_and_linear(orc, T):
    """G(const) = const; G(r) = r at nodes whose gyro-ring does not touch a
    radial boundary (four points average out, bilinear interpolation exact)."""
    cfg, p, g = T
    r, th, ze = _node_coords(p, g)
    out = orc.gyro_op(p, 0, np.full(g.mgrid, 1.75))
    assert np.max(np.abs(out - 1.75)) < 1e-14
    out = orc.gyro_op(p, 1, r[1].copy())
    rhoG = math.sqrt(2) / p.omega0
    inner = (r[1] - rhoG > p.a0) & (r[1] + rhoG < p.a1)
    assert np.max(np.abs(out[inner] - r[1][inner])) < 1e-13


def test_jacobi_small_gyroradius_limit(orc, T):
    """rho_i -> 0: G = I so (1 + 1/tau) phi - phi = rhs gives phi = tau * rhs."""
    cfg, p, g = T
    pp = orc.make_params(dict(cfg, omega0=1e15, poisson_iters=70, tau=1.0))
    rng = np.random.default_rng(3)
    rhs = rng.standard_normal(g.mgrid)
    for i in range(p.mpsi + 1):
        rhs[g.igrid[i] + g.mtheta[i]] = rhs[g.igrid[i]]
    phi = orc.jacobi_plane(pp, 0, rhs)
    inner = np.ones(g.mgrid, bool)
    inner[g.igrid[0]:g.igrid[1]] = False
    inner[g.igrid[p.mpsi]:] = False
    assert np.max(np.abs(phi[inner] - rhs[inner])) < 1e-11
    assert np.all(phi[~inner] == 0)
    assert np.all(orc.jacobi_plane(p, 0, np.zeros(g.mgrid)) == 0)


def test_jacobi_matches_dense_solve(orc, T):
    """Weighted Jacobi converges to the dense LU solution of the assembled
    system (1 + 1/tau) I - G^2 on interior rings (G assembled from unit vectors)."""
    cfg, p, g = T
    pp = orc.make_params(dict(cfg, poisson_iters=60))
    n = g.mgrid
    canon = [g.igrid[i] + j for i in range(1, p.mpsi) for j in range(g.mtheta[i])]

    def expand(v):
        f = np.zeros(n)
        f[canon] = v
        for i in range(p.mpsi + 1):
            f[g.igrid[i] + g.mtheta[i]] = f[g.igrid[i]]
        return f

    A = np.zeros((len(canon), len(canon)))
    for c in range(len(canon)):
        e = np.zeros(len(canon))
        e[c] = 1
        A[:, c] = orc.gyro_op(p, 0, orc.gyro_op(p, 0, expand(e)))[canon]
    A = (1 + 1 / p.tau) * np.eye(len(canon)) - A
    rng = np.random.default_rng(4)
    b = rng.standard_normal(len(canon))
    x = np.linalg.solve(A, b)
    phi = orc.jacobi_plane(pp, 0, expand(b))
    assert np.max(np.abs(phi[canon] - x)) < 1e-10 * np.max(np.abs(x))


def test_field_closed_forms(orc, T):
    cfg, p, g = T
    r, th, ze = _node_coords(p, g)
    K = p.mzetamax
    # constant -> zero gradient
    gp = orc.field(p, np.full((K + 1, g.mgrid), 3.0))
    assert np.max(np.abs(gp)) < 1e-12
    # linear in r -> g_r = 1 exactly (centred and one-sided)
    gp = orc.field(p, r.copy())
    assert np.max(np.abs(gp[..., 0] - 1.0)) < 1e-11
    assert np.max(np.abs(gp[..., 1:])) < 1e-11
    # cos(zeta_k) * c(r): g_par = -sin(zeta_k) sin(dzeta)/dzeta * c(r) exactly
    dz = TWO_PI / K
    c = 1 + r
    gp = orc.field(p, np.cos(ze) * c)
    expect = -np.sin(ze) * math.sin(dz) / dz * c
    assert np.max(np.abs(gp[..., 2] - expect)) < 1e-12


def test_field_theta_derivative_second_order(orc):
    """phi = sin(3 theta_phys): g_theta -> 3 cos(3 theta), error O(dtheta^2)."""
    errs = []
    for mth in (64, 128):
        cfg = synth.config("T", mthetamax=mth)
        p = orc.make_params(cfg)
        g = orc.geometry(p)
        r, th, ze = _node_coords(p, g)
        gp = orc.field(p, np.sin(3 * th))
        inner = r[:p.mzetamax] > 0.5
        errs.append(np.max(np.abs(gp[:p.mzetamax, :, 1][inner] - 3 * np.cos(3 * th[:p.mzetamax][inner]))))
    assert 3.5 < errs[0] / errs[1] < 4.5, errs


def test_poisson_smooth_zero_and_linear(orc, T):
    cfg, p, g = T
    nm = np.ones(p.mpsi + 1)
    z = np.zeros((p.mzetamax + 1, g.mgrid))
    assert np.all(orc.poisson_smooth(p, z, nm) == 0)
    rng = np.random.default_rng(5)
    a = rng.standard_normal(z.shape)
    b = rng.standard_normal(z.shape)
    pa, pb = orc.poisson_smooth(p, a, nm), orc.poisson_smooth(p, b, nm)
    pab = orc.poisson_smooth(p, a + 2 * b, nm)
    assert np.max(np.abs(pab - pa - 2 * pb)) < 1e-10 * np.max(np.abs(pab))
    # Dirichlet: phi = 0 on the boundary rings before the final smooth
    # keeps ring 0 and ring mpsi fixed by the radial smoothing pass
