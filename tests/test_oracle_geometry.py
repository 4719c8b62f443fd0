"""Pins for the oracle's geometry (G-1..G-5) and constants (C-5, C-6).

Pinned against PAPER.md Tab.2, the fig:weakscale caption count
(P:522), the Cyclone constants and the SURVEY G-7 worked table.
"""
import math

import numpy as np
import pytest

import synth
from conftest import golden_path


def _tab2():
    rows, extra = [], {}
    for line in open(golden_path("tab2_grid_sizes.txt")):
        line = line.split("#")[0].split()
        if not line:
            continue
        if len(line) == 2:
            extra[line[0]] = int(line[1])
        else:
            rows.append((line[0], int(line[1]), int(line[2]), int(line[3]), float(line[4]), float(line[5])))
    return rows, extra


@pytest.mark.parametrize("row", _tab2()[0], ids=lambda r: r[0])
def test_mgrid_matches_paper_table2(orc, row):
    size, mpsi, mthetamax, mgrid, chargei, evector = row
    p = orc.make_params(synth.config("a", mpsi=mpsi, mthetamax=mthetamax))
    g = orc.geometry(p)
    assert g.mgrid == mgrid  # exact
    assert int(g.mtheta.astype(np.int64).sum() + len(g.mtheta)) == mgrid
    assert g.mtheta[-1] == mthetamax
    assert np.all(g.mtheta % 2 == 0)
    # chargei / evector rows: MiB for 2 planes of fp64, printed rounding
    digits = 1 if size == "A" else 2
    assert round(mgrid * 2 * 8 / 2**20, digits) == chargei
    assert round(mgrid * 2 * 8 * 3 / 2**20, 2) == evector


def test_particles_per_plane_caption(orc):
    _, extra = _tab2()
    cfg = synth.config("A")
    g = orc.geometry(orc.make_params(cfg))
    assert cfg["micell"] * (g.mgrid - cfg["mpsi"]) == extra["particles_per_plane_A"]


def test_geometry_T_worked_table(orc):
    p = orc.make_params(synth.config("T"))
    g = orc.geometry(p)
    rows = [l.split() for l in open(golden_path("geometry_T.txt")) if l.strip() and not l.startswith("#")]
    for r in rows:
        if r[0] == "mgrid":
            assert g.mgrid == int(r[1])
            continue
        i = int(r[0])
        assert g.mtheta[i] == int(r[2])
        assert g.igrid[i] == int(r[3])
        assert abs(orc.qprofile(p, float(r[1])) - float(r[4])) < 1e-5
        assert g.itran[i] == int(r[5])
        assert abs(g.qtinv[i] - float(r[6])) < 1e-6


def test_cyclone_q_profile(orc):
    p = orc.make_params(synth.config("A"))
    q = orc.qprofile(p, 0.5)
    assert abs(q - 1.4) < 1e-12
    h = 1e-6
    dq = (orc.qprofile(p, 0.5 + h) - orc.qprofile(p, 0.5 - h)) / (2 * h)
    assert abs(0.5 / q * dq - 0.78) < 1e-9  # (r/q) dq/dr = 0.78


def test_gradient_profile(orc):
    assert orc.prof(0.5) == 1.0
    assert abs(orc.prof(0.15) - math.exp(-1)) < 1e-14
    assert abs(orc.prof(0.85) - math.exp(-1)) < 1e-14


def test_equilibrium_field(orc):
    p = orc.make_params(synth.config("A"))
    assert orc.bfield(p, 0.5, math.pi / 2) == pytest.approx(1.0, abs=1e-15)
    assert orc.bfield(p, 0.5, 0.0) == pytest.approx(1.0 / (1.0 + 0.5 / 2.78), rel=1e-15)


def test_seam_rotation_is_field_line(orc):
    """G-4: following a node's label once around the torus lands on node
    (j + itran) of plane 0, i.e. the twist per turn is 2 pi * qtinv ~ 2 pi / q."""
    for size in "TA":
        p = orc.make_params(synth.config(size))
        g = orc.geometry(p)
        r = p.a0 + np.arange(p.mpsi + 1) * (p.a1 - p.a0) / p.mpsi
        q = p.q0 + p.q2 * r * r
        # rationalised twist within half a cell of the analytic one
        assert np.all(np.abs(g.itran - g.mtheta / q) <= 0.5 + 1e-12)
