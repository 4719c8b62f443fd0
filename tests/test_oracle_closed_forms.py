"""Closed-form pins for the parts of the oracle that conservation and
linearity cannot see: the smoothing filter's weights and its seam rotation
(F-4), the gyro-average operator's radius and angular offset (F-1,
P:176), the parallel-gradient seam rotation of the field (F-5, G-4) and
the radial reflection of the push (U-8).  Each expected value is
written from the mathematics, not from the oracle; each test fails for the
matching plausible mistake (weights (1/3,1/3,1/3), rho_G = 1/Omega_0,
theta +- rho_G instead of theta +- rho_G/r, the seam rotation dropped,
reflection replaced by clamping)."""
import math

import numpy as np
import pytest

import synth

TWO_PI = 2 * math.pi


def _ring(g, i):
    return slice(int(g.igrid[i]), int(g.igrid[i]) + int(g.mtheta[i]))


def _phys_theta(p, g, k, i):
    """Physical angle of the canonical nodes of ring i on plane k (G-4)."""
    j = np.arange(g.mtheta[i])
    return j * TWO_PI / g.mtheta[i] + k * TWO_PI / p.mzetamax * g.qtinv[i]


# ---------------------------------------------------------------- F-4 smooth
@pytest.mark.parametrize("K,m", [(2, 3), (4, 3), (4, 2), (6, 1)])
def test_smooth_theta_mode_and_parallel_seam(orc, K, m):
    """Input: cos(2 pi m j / mt_0) on ring 0 of every plane, zero elsewhere.
    The theta pass (1/4, 1/2, 1/4) multiplies a ring Fourier mode by exactly
    A = 1/2 + 1/2 cos(2 pi m / mt_0); the radial pass keeps the boundary ring
    0; the parallel pass (1/4, 1/2, 1/4) at fixed label leaves the
    plane-independent mode unchanged on interior planes, while planes 0 and
    K-1 see their neighbour across the seam rotated by itran_0 nodes
    (node(K, j) == node(0, j + itran), G-4):
      k = 0:   A (3/4 cos x_j + 1/4 cos x_{j - itran})
      k = K-1: A (3/4 cos x_j + 1/4 cos x_{j + itran})."""
    cfg = synth.config("T", mzetamax=K)
    p = orc.make_params(cfg)
    g = orc.geometry(p)
    mt, it = int(g.mtheta[0]), int(g.itran[0])
    assert (m * it) % mt != 0  # the seam rotation is visible for this mode
    f = np.zeros((K + 1, g.mgrid))
    j = np.arange(mt + 1)
    for k in range(K):
        f[k, int(g.igrid[0]):int(g.igrid[0]) + mt + 1] = np.cos(TWO_PI * m * j / mt)
    f[K] = 0.0  # the seam plane is rebuilt by the oracle from plane 0
    out = orc.smooth(p, f)
    A = 0.5 + 0.5 * math.cos(TWO_PI * m / mt)
    jj = np.arange(mt)
    x = lambda s: np.cos(TWO_PI * m * ((jj + s) % mt) / mt)  # noqa: E731
    for k in range(K):
        want = A * x(0)
        if k == 0:
            want = A * (0.75 * x(0) + 0.25 * x(-it))
        if k == K - 1:
            want = A * (0.75 * x(0) + 0.25 * x(+it))
        got = out[k, _ring(g, 0)]
        assert np.max(np.abs(got - want)) < 1e-14, (k, np.max(np.abs(got - want)))


def test_smooth_radial_pass_quadratic(orc):
    """f = r^2 (ring-constant, plane-constant): the theta and parallel passes
    leave it unchanged; the radial pass (1/4, 1/2, 1/4) gives exactly
    r^2 + dr^2/2 on interior rings (ring-constant values interpolate exactly)
    and keeps the boundary rings."""
    cfg = synth.config("T", mzetamax=4)
    p = orc.make_params(cfg)
    g = orc.geometry(p)
    dr = (p.a1 - p.a0) / p.mpsi
    f = np.zeros((p.mzetamax + 1, g.mgrid))
    for i in range(p.mpsi + 1):
        f[:, int(g.igrid[i]):int(g.igrid[i + 1])] = (p.a0 + i * dr) ** 2
    out = orc.smooth(p, f)
    for i in range(p.mpsi + 1):
        r = p.a0 + i * dr
        want = r * r if i in (0, p.mpsi) else r * r + 0.5 * dr * dr
        assert np.max(np.abs(out[:p.mzetamax, _ring(g, i)] - want)) < 1e-15


# ---------------------------------------------------------------- F-1 gyro operator
def _gyro_mode_error(orc, mthetamax, m):
    cfg = synth.config("T", mthetamax=mthetamax, mzetamax=2)
    p = orc.make_params(cfg)
    g = orc.geometry(p)
    rhoG = math.sqrt(2.0) / p.omega0
    dr = (p.a1 - p.a0) / p.mpsi
    f = np.zeros(g.mgrid)
    for i in range(p.mpsi + 1):
        th = np.arange(g.mtheta[i] + 1) * TWO_PI / g.mtheta[i]
        f[int(g.igrid[i]):int(g.igrid[i + 1])] = np.cos(m * th)
    out = orc.gyro_op(p, 0, f)
    err = 0.0
    for i in range(p.mpsi + 1):
        r = p.a0 + i * dr
        if r - rhoG < p.a0 or r + rhoG > p.a1:
            continue
        th = _phys_theta(p, g, 0, i)
        want = np.cos(m * th) * (0.5 + 0.5 * math.cos(m * rhoG / r))
        err = max(err, float(np.max(np.abs(out[_ring(g, i)] - want))))
    return err


def test_gyro_op_fourier_mode_converges_to_bessel_like_factor(orc):
    """G cos(m theta) -> cos(m theta) [1/2 + 1/2 cos(m rho_G / r)], rho_G =
    sqrt(2)/Omega_0 (F-1): the two radial points see cos(m theta) unchanged,
    the two angular points at theta +- rho_G/r give cos(m theta) cos(m rho_G/r).
    Linear label interpolation errs by O((m dtheta)^2): second-order
    convergence under mthetamax refinement."""
    m = 5
    errs = [_gyro_mode_error(orc, mth, m) for mth in (256, 512, 1024, 2048)]
    for a, b in zip(errs, errs[1:]):
        assert 3.3 < a / b < 4.7, errs
    assert errs[-1] < 5e-4, errs


def test_gyro_op_radial_points_quadratic(orc):
    """G r^2 = 1/4 [(r + rho_G)^2 + (r - rho_G)^2 + 2 r^2] = r^2 + rho_G^2/2 at
    nodes away from the boundaries, up to the linear radial interpolation
    error (x - r_i)(r_{i+1} - x) in [0, dr^2/4] of each radial point; Omega_0
    fixed while the rings are refined (mpsi 128: dr^2/8 = 5e-6 << rho_G^2/2 =
    2e-3)."""
    cfg = synth.config("T", mpsi=128, mthetamax=256, mzetamax=2, omega0=22.0)
    p = orc.make_params(cfg)
    g = orc.geometry(p)
    dr = (p.a1 - p.a0) / p.mpsi
    rhoG = math.sqrt(2.0) / p.omega0
    f = np.zeros(g.mgrid)
    for i in range(p.mpsi + 1):
        f[int(g.igrid[i]):int(g.igrid[i + 1])] = (p.a0 + i * dr) ** 2
    out = orc.gyro_op(p, 0, f)
    n = 0
    for i in range(p.mpsi + 1):
        r = p.a0 + i * dr
        if r - rhoG < p.a0 or r + rhoG > p.a1:
            continue
        d = out[_ring(g, i)] - (r * r + 0.5 * rhoG * rhoG)
        assert np.all(d >= -1e-15) and np.all(d <= dr * dr / 8 + 1e-15), (i, d.min(), d.max())
        n += 1
    assert n > 100


# ---------------------------------------------------------------- F-5 field
def _field_par_error(orc, K, n, l):
    cfg = synth.config("T", mzetamax=K)
    p = orc.make_params(cfg)
    g = orc.geometry(p)
    phi = np.zeros((K + 1, g.mgrid))
    for k in range(K + 1):
        for i in range(p.mpsi + 1):
            th = np.arange(g.mtheta[i] + 1) * TWO_PI / g.mtheta[i] + k * TWO_PI / K * g.qtinv[i]
            phi[k, int(g.igrid[i]):int(g.igrid[i + 1])] = np.cos(n * th - l * k * TWO_PI / K)
    gp = orc.field(p, phi)
    err = np.zeros(K)
    for k in range(K):
        for i in range(p.mpsi + 1):
            th = _phys_theta(p, g, k, i)
            want = -(n * g.qtinv[i] - l) * np.sin(n * th - l * k * TWO_PI / K)
            err[k] = max(err[k], float(np.max(np.abs(gp[k, _ring(g, i), 2] - want))))
    return err


def test_field_parallel_gradient_through_the_seam(orc):
    """phi = cos(n theta - l zeta) on the field-aligned grid: along a field line
    (fixed label, theta = alpha + zeta qtinv_i) d phi/d zeta = -(n qtinv_i - l)
    sin(n theta - l zeta).  The centred difference across planes converges at
    second order on every plane, including 0 and K-1 whose neighbour lies
    across the seam (node(K, j) == node(0, j + itran), G-4)."""
    e32 = _field_par_error(orc, 32, 3, 1)
    e64 = _field_par_error(orc, 64, 3, 1)
    assert np.all(e64 < 0.025), e64  # amplitude n qtinv - l up to 2.4
    # second order on every plane (same zeta: plane k of 32 = plane 2k of 64),
    # the seam planes 0 and K-1 included
    ratio = e32 / e64[::2]
    assert np.all((ratio > 3.6) & (ratio < 4.4)), ratio
    assert 3.6 < e32[31] / e64[63] < 4.4


def test_field_radial_gradient_at_physical_angle(orc):
    """phi = r cos(theta): g_r = d phi/dr at fixed physical theta = cos(theta)
    (neighbour rings interpolated at the node's physical angle, F-5); exact in
    r, O(dtheta^2) from the label interpolation -> second-order convergence."""
    def err(mth):
        cfg = synth.config("T", mthetamax=mth, mzetamax=2)
        p = orc.make_params(cfg)
        g = orc.geometry(p)
        dr = (p.a1 - p.a0) / p.mpsi
        phi = np.zeros((3, g.mgrid))
        for k in range(3):
            for i in range(p.mpsi + 1):
                th = np.arange(g.mtheta[i] + 1) * TWO_PI / g.mtheta[i] + k * TWO_PI / 2 * g.qtinv[i]
                phi[k, int(g.igrid[i]):int(g.igrid[i + 1])] = (p.a0 + i * dr) * np.cos(th)
        gp = orc.field(p, phi)
        e = 0.0
        for k in range(2):
            for i in range(p.mpsi + 1):
                e = max(e, float(np.max(np.abs(gp[k, _ring(g, i), 0] - np.cos(_phys_theta(p, g, k, i))))))
        return e
    e = [err(m) for m in (256, 512, 1024)]
    assert 3.3 < e[0] / e[1] < 4.7 and 3.3 < e[1] / e[2] < 4.7, e
    assert e[-1] < 1e-3


# ---------------------------------------------------------------- U-8 reflection
@pytest.mark.parametrize("edge", ["outer", "inner"])
def test_push_reflection_closed_form(orc, edge):
    """A marker that crosses r = a1 (or a0) in one stage comes back at
    r' = 2 a1 - r (or 2 a0 - r), psi' = r'^2 / 2, with theta, zeta, rho_par, w
    those of the unreflected update X + h F(X) (U-7, U-8).  The
    vertical curvature drift v_d,r = -C_d sin(theta) moves the marker outward
    at theta = 3 pi/2 and inward at theta = pi/2 (field off)."""
    cfg = synth.config("T")
    p = orc.make_params(cfg)
    h = 0.5 * p.dt
    vpar, mu = 3.0, 0.5
    if edge == "outer":
        r0, th0 = p.a1 - 0.002, 1.5 * math.pi
    else:
        r0, th0 = p.a0 + 0.002, 0.5 * math.pi
    B = 1.0 / (1.0 + r0 / p.R0 * math.cos(th0))
    X = np.array([0.5 * r0 * r0, th0, 0.3, vpar / (p.omega0 * B), 0.01])
    F = orc.rhs(p, X, mu, np.zeros(3))
    x = X + h * F
    rn = math.sqrt(2 * x[0])
    assert (rn > p.a1) if edge == "outer" else (rn < p.a0)
    rr = 2 * p.a1 - rn if edge == "outer" else 2 * p.a0 - rn
    Xa = {k: np.array([X[d]]) for d, k in enumerate(orc.ATTRS)}
    Xb = {k: v.copy() for k, v in Xa.items()}
    g = orc.geometry(p)
    gp = np.zeros((p.mzetamax + 1, g.mgrid, 3))
    nrefl = orc.push(p, 1, Xa, Xb, np.array([mu]), gp)
    assert nrefl == 1
    assert abs(Xb["psi"][0] - 0.5 * rr * rr) <= 1e-15
    assert abs(Xb["rho"][0] - x[3]) <= 1e-15 and abs(Xb["w"][0] - x[4]) <= 1e-15
    assert abs(Xb["theta"][0] - (x[1] % TWO_PI)) <= 1e-15 and abs(Xb["zeta"][0] - x[2]) <= 1e-15
