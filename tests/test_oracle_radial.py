"""Pins for the oracle's radial decomposition functions: G-6 equal-area
windows snapped to rings and H-2 radial destination (P:244-249,
SPEC S:553).  Pinned against values computed independently of the oracle
(SURVEY §8(c) G-6 [computed]) and an exact-decimal brute force."""
from decimal import Decimal, getcontext

import numpy as np

import synth

getcontext().prec = 60


def _exact_bounds(cfg, K):
    """Exact-decimal equal-area radii r_k = sqrt(a0^2 + (k/K)(a1^2 - a0^2)),
    snapped to the nearest ring index (no half-way ties occur in the presets)."""
    a0, a1, M = Decimal(cfg["a0"]), Decimal(cfg["a1"]), cfg["mpsi"]
    dr = (a1 - a0) / M
    out = [0]
    for k in range(1, K):
        rk = (a0 * a0 + Decimal(k) / K * (a1 * a1 - a0 * a0)).sqrt()
        x = (rk - a0) / dr
        assert abs(x - x.to_integral_value() - Decimal("0.5")) > Decimal("1e-6")  # no tie
        out.append(int((x + Decimal("0.5")).to_integral_value(rounding="ROUND_FLOOR")))
    out.append(M)
    return out


def test_radial_windows_class_D_split_ring_519(orc):
    """SURVEY G-6 [computed]: class D (mpsi 768, mthetamax 5632) at K = 2 splits
    at ring 519; owned sum(mtheta) 1,201,004 (rings 0..518) and 1,205,110
    (rings 519..768); 0.3 % imbalance."""
    p = orc.make_params(synth.config("D"))
    g = orc.geometry(p)
    b = orc.radial_windows(p, 2)
    assert list(b) == [0, 519, 768]
    assert int(g.mtheta[0:519].sum()) == 1201004
    assert int(g.mtheta[519:769].sum()) == 1205110


def test_radial_windows_match_exact_decimal(orc):
    for size in "TABCD":
        cfg = synth.config(size)
        p = orc.make_params(cfg)
        for K in (1, 2, 3, 4, 8):
            assert list(orc.radial_windows(p, K)) == _exact_bounds(cfg, K), (size, K)


def test_radial_windows_equal_area(orc):
    """Each window's annulus area differs from 1/K of the total by at most the
    area of one ring spacing at the outer edge (snapping moves a boundary by
    <= dr/2)."""
    for size in "ABCD":
        cfg = synth.config(size)
        p = orc.make_params(cfg)
        dr = (p.a1 - p.a0) / p.mpsi
        for K in (2, 4, 8):
            b = orc.radial_windows(p, K)
            r = p.a0 + b * dr
            area = np.diff(r ** 2)
            tot = p.a1 ** 2 - p.a0 ** 2
            assert np.all(np.abs(area - tot / K) <= 2 * p.a1 * dr + 1e-15), (size, K)


def test_radial_dest_brute_force(orc):
    """Owner window = the k with r(bound_k) <= sqrt(2 psi) < r(bound_k+1),
    evaluated in exact decimal arithmetic on the fp64 psi and the fp64 ring
    radii (particles within 1e-12 of a boundary are skipped: there fp64
    rounding of the sqrt decides)."""
    cfg = synth.config("D")
    p = orc.make_params(cfg)
    rng = np.random.default_rng(3)
    r = p.a0 + (p.a1 - p.a0) * rng.random(6000)
    psi = 0.5 * r * r
    dr = (p.a1 - p.a0) / p.mpsi
    for K in (2, 4, 8):
        b = orc.radial_windows(p, K)
        dest = orc.radial_dest(p, psi, K)
        rb = [Decimal(float(p.a0 + int(x) * dr)) for x in b]
        for ps, d in zip(psi, dest):
            re = (2 * Decimal(float(ps))).sqrt()
            if min(abs(re - x) for x in rb[1:K]) < Decimal("1e-12"):
                continue
            want = sum(1 for x in rb[1:K] if re >= x)
            assert d == want
        assert dest.min() >= 0 and dest.max() == K - 1


def test_radial_dest_edges(orc):
    """A particle exactly on a boundary ring belongs to the outer window; r = a0
    to window 0; r = a1 to the last window."""
    p = orc.make_params(synth.config("D"))
    dr = (p.a1 - p.a0) / p.mpsi
    rb = p.a0 + 519 * dr
    psi = np.array([0.5 * p.a0 ** 2, 0.5 * p.a1 ** 2, 0.5 * rb * rb, 0.5 * np.nextafter(rb, 0) ** 2])
    d = orc.radial_dest(p, psi, 2)
    r_back = np.sqrt(2 * psi)
    assert d[0] == 0 and d[1] == 1
    assert d[2] == (1 if r_back[2] >= rb else 0)
    assert d[3] == 0
