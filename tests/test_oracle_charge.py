"""Pins for the oracle's charge deposition and reductions (Q-1..Q-8), and
gather (U-2): conservation, hand cases, brute-force node-centric deposit,
unique-node counts, adjointness, special cases."""
import math

import numpy as np
import pytest

import synth
from conftest import golden_path

TWO_PI = 2 * math.pi


@pytest.fixture(scope="module")
def T(orc):
    cfg = synth.config("T")
    p = orc.make_params(cfg)
    return cfg, p, orc.geometry(p)


def _one(psi, theta, zeta, mu, w=1.0):
    return dict(psi=np.array([psi]), theta=np.array([theta]), zeta=np.array([zeta]),
                mu=np.array([mu]), w=np.array([w]))


def test_charge_conservation(orc, T):
    """Sum of deposited charge equals the sum of weights (P:202 partition of
    unity; clamping keeps it exact).  Normalised by sum|w| (mixed signs)."""
    cfg, p, g = T
    parts = synth.load_particles(cfg, 12100, seed=1)
    grid, nclamp = orc.deposit(p, parts)
    assert nclamp == 0
    sw, saw = parts["w"].sum(), np.abs(parts["w"]).sum()
    assert abs(grid.sum() - sw) <= 1e-12 * saw
    red = orc.charge_reduce_global(p, grid)
    canon = sum(red[k, g.igrid[i]:g.igrid[i] + g.mtheta[i]].sum() for k in range(p.mzetamax) for i in range(p.mpsi + 1))
    assert abs(canon - sw) <= 1e-12 * saw


def test_charge_hand_cases(orc, T):
    cfg, p, g = T
    lines = [l for l in open(golden_path("charge_hand_cases.txt")) if l.strip() and not l.startswith("#")]
    cases, cur = [], None
    for l in lines:
        t = l.split()
        if t[0].startswith("case"):
            cur = dict(zeta=float(t[1]) * math.pi, theta=float(t[2]) * math.pi, exp=[])
            cases.append(cur)
        else:
            cur["exp"].append((int(t[0]), int(t[1]), int(t[2]), float(t[3])))
    for c in cases:
        grid, _ = orc.deposit(p, _one(0.5 * 0.35 ** 2, c["theta"], c["zeta"], 0.0))
        red = orc.charge_reduce_global(p, grid)
        canon = np.zeros_like(red[:p.mzetamax])
        for k in range(p.mzetamax):
            for i in range(p.mpsi + 1):
                canon[k, g.igrid[i]:g.igrid[i] + g.mtheta[i]] = red[k, g.igrid[i]:g.igrid[i] + g.mtheta[i]]
        expect = np.zeros_like(canon)
        for k, i, j, v in c["exp"]:
            expect[k, g.igrid[i] + j] = v
        assert np.max(np.abs(canon - expect)) < 1e-14


def _brute_force(cfg, g, parts):
    """Node-centric deposit written from the hat-function definition: each node
    (plane kk, ring m, label j) receives w/4 * sum_l hat(x_l - m) * hat_per(s_lm - j)
    * hat(t_g - kk), with x_l the clamped radial cell coordinate, s_lm the label
    coordinate on ring m (periodic distance), t_g = zeta*mzetamax/(2 pi)."""
    K, mpsi = cfg["mzetamax"], cfg["mpsi"]
    a0, a1 = cfg["a0"], cfg["a1"]
    dr = (a1 - a0) / mpsi
    out = np.zeros((K + 1, g.mgrid))
    hat = lambda x: max(0.0, 1.0 - abs(x))
    for ip in range(len(parts["w"])):
        r = math.sqrt(2 * parts["psi"][ip])
        th, ze, mu, w = parts["theta"][ip], parts["zeta"][ip], parts["mu"][ip], parts["w"][ip]
        B = 1.0 / (1.0 + r / cfg["R0"] * math.cos(th))
        rho = math.sqrt(2 * mu / B) / cfg["omega0"]
        tg = ze * K / TWO_PI
        pts = [(r + rho, th), (r, th + rho / r), (r - rho, th), (r, th - rho / r)]
        for (rl, tl) in pts:
            x = (min(max(rl, a0), a1) - a0) / dr
            for m in range(mpsi + 1):
                hr = hat(x - m)
                if hr == 0.0:
                    continue
                mt = int(g.mtheta[m])
                s = ((tl - ze * g.qtinv[m]) / TWO_PI % 1.0) * mt
                for j in range(mt):
                    d = abs(s - j) % mt
                    d = min(d, mt - d)
                    ht = hat(d)
                    if ht == 0.0:
                        continue
                    for kk in range(K + 1):
                        hz = hat(tg - kk)
                        if hz:
                            out[kk, g.igrid[m] + j] += 0.25 * w * hr * ht * hz
    return out


def test_charge_brute_force(orc, T):
    cfg, p, g = T
    parts = synth.load_particles(cfg, 40, seed=7, w_amp=1.0)
    # include edge cases: a gyro-ring clamped at both radial boundaries, zeta at 0
    parts["psi"][0] = 0.5 * 0.101 ** 2
    parts["mu"][0] = 4.0
    parts["psi"][1] = 0.5 * 0.899 ** 2
    parts["mu"][1] = 4.0
    parts["zeta"][2] = 0.0
    grid, _ = orc.deposit(p, parts)
    folded = grid.copy()
    for k in range(p.mzetamax + 1):
        for i in range(p.mpsi + 1):
            folded[k, g.igrid[i]] += folded[k, g.igrid[i] + g.mtheta[i]]
            folded[k, g.igrid[i] + g.mtheta[i]] = 0.0
    bf = _brute_force(cfg, g, parts)
    assert np.max(np.abs(folded - bf)) <= 1e-13 * np.abs(parts["w"]).sum()


def test_unique_nodes_8_to_32(orc, T):
    """a particle deposits onto as few as 8 and as many as 32 nodes."""
    cfg, p, g = T
    parts = synth.load_particles(cfg, 200, seed=3)
    counts = []
    for ip in range(200):
        one = {k: parts[k][ip:ip + 1] for k in ("psi", "theta", "zeta", "mu", "w")}
        grid, _ = orc.deposit(p, one, w=np.ones(1))
        counts.append(int((grid != 0).sum()))
    assert min(counts) >= 8 and max(counts) <= 32
    # mu = 0 -> the four points coincide -> exactly 8 nodes (generic position)
    grid, _ = orc.deposit(p, _one(0.5 * 0.4321 ** 2, 1.2345, 0.777, 0.0))
    assert int((grid != 0).sum()) == 8


def test_marker_norm_conservation(orc, T):
    cfg, p, g = T
    parts = synth.load_particles(cfg, 5000, seed=11)
    nm = orc.marker_norm(p, parts)
    total = sum(nm[i] * p.mzetamax * g.mtheta[i] for i in range(p.mpsi + 1))
    assert abs(total - 5000) < 1e-9


def _field_consistent(p, g, rng, ncomp=3):
    """Random field with duplicates and the seam plane consistent (G-2, G-4)."""
    K = p.mzetamax
    f = rng.standard_normal((K + 1, g.mgrid, ncomp))
    for k in range(K):
        for i in range(p.mpsi + 1):
            f[k, g.igrid[i] + g.mtheta[i]] = f[k, g.igrid[i]]
    for i in range(p.mpsi + 1):
        for j in range(g.mtheta[i] + 1):
            f[K, g.igrid[i] + j] = f[0, g.igrid[i] + (j + g.itran[i]) % g.mtheta[i]]
    return f


def test_gather_constant_field(orc, T):
    cfg, p, g = T
    parts = synth.load_particles(cfg, 300, seed=5)
    gp = np.zeros((p.mzetamax + 1, g.mgrid, 3))
    gp[..., 0], gp[..., 1], gp[..., 2] = 0.3, -1.7, 2.5
    gb = orc.gather(p, parts, gp)
    assert np.max(np.abs(gb - np.array([0.3, -1.7, 2.5]))) < 1e-14


def test_gather_adjoint_of_deposit(orc, T):
    """<deposit(w), g> == <w, gather(g)> (SPEC S:427 adjointness)."""
    cfg, p, g = T
    rng = np.random.default_rng(0)
    parts = synth.load_particles(cfg, 500, seed=9, w_amp=1.0)
    f = _field_consistent(p, g, rng)
    grid, _ = orc.deposit(p, parts)
    lhs = (grid * f[..., 1]).sum()
    rhs = (parts["w"] * orc.gather(p, parts, f)[:, 1]).sum()
    assert abs(lhs - rhs) < 1e-12 * max(1.0, abs(lhs))


def test_gather_mu0_at_node(orc, T):
    cfg, p, g = T
    rng = np.random.default_rng(1)
    f = _field_consistent(p, g, rng)
    i, j = 7, 5
    r = p.a0 + i * (p.a1 - p.a0) / p.mpsi
    zeta = 0.0
    theta = j * TWO_PI / g.mtheta[i]
    gb = orc.gather(p, _one(0.5 * r * r, theta, zeta, 0.0), f)
    assert np.max(np.abs(gb[0] - f[0, g.igrid[i] + j])) < 1e-9


def test_marker_norm_node_markers_closed_form(orc, T):
    """Q-8 pinned by hand: markers with mu = 0 (the four gyro-points coincide)
    sitting on grid nodes (r = r_i, zeta on a plane, theta on a field-line
    label) each deposit exactly one unit on their own ring, so the marker
    density of ring i is (markers on ring i) / (mzetamax * mtheta_i): the mean
    over the mzetamax planes and the mtheta_i canonical nodes (not mtheta_i + 1
    with the duplicate, nor mzetamax + 1 planes with the seam copy)."""
    cfg, p, g = T
    rng = np.random.default_rng(12)
    K, M = p.mzetamax, p.mpsi
    dr = (p.a1 - p.a0) / M
    cnt = np.zeros(M + 1)
    psi, theta, zeta = [], [], []
    for i in range(M + 1):
        for _ in range(i % 5 + 1):
            k = int(rng.integers(K))
            j = int(rng.integers(g.mtheta[i]))
            z = k * 2 * math.pi / K
            r = p.a0 + i * dr
            psi.append(0.5 * r * r)
            zeta.append(z)
            theta.append((2 * math.pi * j / g.mtheta[i] + z * g.qtinv[i]) % (2 * math.pi))
            cnt[i] += 1
    parts = dict(psi=np.array(psi), theta=np.array(theta), zeta=np.array(zeta), mu=np.zeros(len(psi)))
    nm = orc.marker_norm(p, parts)
    expect = cnt / (K * np.asarray(g.mtheta[:M + 1], dtype=float))
    assert np.allclose(nm, expect, rtol=0, atol=1e-12 * expect.max())
