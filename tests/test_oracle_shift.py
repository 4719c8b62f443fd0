"""Pins for the oracle's shift destination (H-1) and bin key (H-4)."""
import math
from decimal import Decimal, getcontext

import numpy as np
import pytest

import synth

getcontext().prec = 60
PI = Decimal("3.14159265358979323846264338327950288419716939937510582097494")


def test_shift_dest_brute_force(orc):
    """Destination domain = the domain whose planes bracket zeta, computed with
    exact decimal arithmetic on the fp64 zeta value (boundaries within 1e-12
    of a plane are skipped: there fp64 rounding decides)."""
    cfg = synth.config("A")
    p = orc.make_params(cfg)
    rng = np.random.default_rng(0)
    zeta = rng.random(20000) * 2 * math.pi
    for P in (64, 32, 16, 8):
        dest = orc.shift_dest(p, zeta, P)
        for z, d in zip(zeta[:4000], dest[:4000]):
            t = Decimal(float(z)) * p.mzetamax / (2 * PI)
            kg = min(int(t), p.mzetamax - 1)
            if abs(t - round(t)) < Decimal("1e-12"):
                continue
            assert d == kg // P
        assert dest.min() >= 0 and dest.max() < p.mzetamax // P


def test_shift_dest_edges(orc):
    p = orc.make_params(synth.config("A"))
    z = np.array([0.0, np.nextafter(2 * math.pi, 0), 2 * math.pi * 0.5])
    d = orc.shift_dest(p, z, 8)
    assert d[0] == 0 and d[1] == 7 and d[2] == 4


def test_bin_key_cell_centres(orc):
    """A gyrocentre placed at the centre of cell (ring i, label cell c, plane
    interval k) gets key (igrid_i + c) * P + k."""
    cfg = synth.config("T")
    p = orc.make_params(cfg)
    g = orc.geometry(p)
    K = p.mzetamax
    dr = (p.a1 - p.a0) / p.mpsi
    rows = []
    for i in range(p.mpsi):
        for c in range(g.mtheta[i]):
            for k in range(K):
                zeta = (k + 0.5) * 2 * math.pi / K
                r = p.a0 + (i + 0.5) * dr
                theta = ((c + 0.5) * 2 * math.pi / g.mtheta[i] + zeta * g.qtinv[i]) % (2 * math.pi)
                rows.append((0.5 * r * r, theta, zeta, (g.igrid[i] + c) * K + k))
    a = np.array(rows)
    parts = dict(psi=a[:, 0], theta=a[:, 1], zeta=a[:, 2])
    key = orc.bin_key(p, parts)
    assert np.array_equal(key, a[:, 3].astype(np.int64))


def test_bin_key_mu_subbins_refine_the_cell_key(orc):
    """H-4 with nmu magnetic-moment sub-bins: key // nmu is the plain cell key,
    the sub-bin is monotone in mu, and for mu ~ Exp(1) (the loader's
    v_perp^2 / 2B at B = 1) each of the nmu quantile bins holds 1/nmu of the
    markers."""
    cfg = synth.config("T")
    p = orc.make_params(cfg)
    parts = synth.load_particles(cfg, 20000, seed=5)
    rng = np.random.default_rng(11)
    parts["mu"] = rng.exponential(1.0, len(parts["psi"]))
    k1 = orc.bin_key(p, parts)
    for nmu in (2, 4, 8):
        kn = orc.bin_key(p, parts, nmu=nmu)
        assert np.array_equal(kn // nmu, k1)
        b = kn % nmu
        frac = np.bincount(b, minlength=nmu) / len(b)
        assert np.all(np.abs(frac - 1.0 / nmu) < 0.02), frac
        order = np.argsort(parts["mu"])
        same = {k: np.repeat(parts[k][:1], len(order)) for k in ("psi", "theta", "zeta")}
        same["mu"] = parts["mu"][order]
        bs = orc.bin_key(p, same, nmu=nmu) % nmu
        assert np.all(np.diff(bs) >= 0)
