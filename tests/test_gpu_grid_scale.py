"""Grid-kernel parity at the configs' geometries (SURVEY §8(a) a7 at scale):
poisson_smooth (F-1..F-4) and field (F-5) of the CUDA path
against the oracle on the class-A grid (32,449 nodes/plane) and the class-D
grid (2,406,883 nodes/plane: the host-built PoisRing constants and label maps
at 769 rings), with few planes and -- at D -- fewer Jacobi sweeps so that the
single-threaded oracle finishes in seconds (both sides use the same count).
Plus one full step (two RK2 stages, every kernel of the path) at D geometry
with the fp32 state (precision 32, tolerance 1e-4)."""
import math

import numpy as np
import pytest

import synth
from test_gpu_parity import G, TOL, ctx_for, rel_err, circ  # noqa: F401

pytestmark = pytest.mark.gpu
TWO_PI = 2 * math.pi

# T with 3 planes: an odd plane count (the gyro-average kernels do 2 planes
# per thread, the last group has one)
GEOMS = [("A", dict(mzetamax=4)), ("D", dict(mzetamax=2, poisson_iters=3)), ("T", dict(mzetamax=3))]


def _charge_input(orc, cfg, p, n, seed):
    parts = synth.load_particles(cfg, n, seed=seed, w_amp=0.1)
    return parts, orc.charge_global(p, parts), orc.marker_norm(p, parts)


@pytest.mark.parametrize("size,over", GEOMS, ids=[g[0] + str(g[1]["mzetamax"]) for g in GEOMS])
def test_poisson_smooth_parity_at_scale(G, orc, size, over):
    cfg = synth.config(size, **over)
    p = orc.make_params(cfg)
    parts, charge, nm = _charge_input(orc, cfg, p, 200_000, 21)
    ctx = ctx_for(G, size, **over)
    ctx.set_grid(G.GRID_CHARGE, charge)
    ctx.set_grid(G.GRID_MARKER, nm)
    ctx.poisson_smooth()
    got = ctx.get_grid(G.GRID_PHI)
    ref = orc.poisson_smooth(p, charge, nm)
    assert got.shape == ref.shape
    assert rel_err(got, ref) <= TOL
    ctx.close()


@pytest.mark.parametrize("size,over", GEOMS, ids=[g[0] + str(g[1]["mzetamax"]) for g in GEOMS])
def test_field_parity_at_scale(G, orc, size, over):
    """Gradient of a potential with structure on every ring and plane (a
    drift-wave-like mode plus noise, smoothed), through the seam."""
    cfg = synth.config(size, **over)
    p = orc.make_params(cfg)
    g = orc.geometry(p)
    K = p.mzetamax
    rng = np.random.default_rng(5)
    phi = np.zeros((K + 1, g.mgrid))
    dr = (p.a1 - p.a0) / p.mpsi
    for k in range(K + 1):
        for i in range(p.mpsi + 1):
            th = np.arange(g.mtheta[i] + 1) * TWO_PI / g.mtheta[i] + k * TWO_PI / K * g.qtinv[i]
            r = p.a0 + i * dr
            phi[k, int(g.igrid[i]):int(g.igrid[i + 1])] = math.sin(9 * r) * np.cos(7 * th - 2 * k * TWO_PI / K)
    phi += 1e-2 * rng.standard_normal(phi.shape)
    ctx = ctx_for(G, size, **over)
    ctx.set_grid(G.GRID_PHI, phi)
    ctx.field()
    got = ctx.get_grid(G.GRID_GRADPHI)
    ref = orc.field(p, phi)
    assert rel_err(got, ref) <= TOL
    ctx.close()


def test_one_step_parity_D_geometry_fp32(G, orc):
    """Class-D geometry, fp32 particle state, ~200 k markers on 2 planes: one
    full step (charge, poisson_smooth, field, push, shift/bin, twice) against
    the oracle's step on the same fp32-rounded markers."""
    over = dict(mzetamax=2, poisson_iters=3)
    cfg = synth.config("D", **over)
    p = orc.make_params(cfg)
    parts = synth.load_particles(cfg, 200_000, seed=31)
    for k in ("psi", "theta", "zeta", "rho", "w", "mu"):
        parts[k] = parts[k].astype(np.float32).astype(np.float64)
    for k in ("theta", "zeta"):
        parts[k] = np.where(parts[k] >= TWO_PI, 0.0, parts[k])
    nm = orc.marker_norm(p, parts)
    ctx = G.Context(G.gtcp_default_params("D", track_ids=1, precision=32, bin_every=1, **over))
    ctx.set_particles(parts)
    assert rel_err(ctx.get_grid(G.GRID_MARKER), nm) <= 1e-4
    ctx.set_grid(G.GRID_MARKER, nm)
    ctx.step(1)
    got = ctx.get_particles()
    ref = {k: v.copy() for k, v in parts.items()}
    orc.step_global(p, ref, nm)
    o1, o2 = np.argsort(got["id"]), np.argsort(ref["id"])
    assert np.array_equal(got["id"][o1], ref["id"][o2])
    for k in ("psi", "rho", "w"):
        assert rel_err(got[k][o1], ref[k][o2]) <= 1e-4, k
    for k in ("theta", "zeta"):
        assert float(np.max(np.abs(circ(got[k][o1], ref[k][o2])))) / TWO_PI <= 1e-4, k
    ctx.close()
