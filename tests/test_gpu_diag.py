"""Diagnostics (gtcp_diag; SPEC S:578-586 history record): heat flux and field
energy against the oracle on the same prescribed potential and gradient field,
and the ITG workload's qualitative behaviour (SPEC acceptance
11): exponential field-energy growth followed by saturation."""
import math
import os
import sys

import numpy as np
import pytest

import synth
from test_gpu_parity import G, ctx_for, rel_err  # noqa: F401

pytestmark = pytest.mark.gpu
TWO_PI = 2 * math.pi


def test_diag_parity_prescribed_field(G, orc):
    cfg = synth.config("T")
    p = orc.make_params(cfg)
    g = orc.geometry(p)
    parts = synth.load_particles(cfg, 12100, seed=41, w_amp=0.1)
    rng = np.random.default_rng(7)
    phi = orc.smooth(p, rng.standard_normal((p.mzetamax + 1, g.mgrid)))
    gp = orc.field(p, phi)
    ctx = ctx_for(G, "T")
    ctx.set_particles(parts)
    ctx.set_grid(G.GRID_PHI, phi)
    ctx.set_grid(G.GRID_GRADPHI, gp)
    d = ctx.diag()
    q_ref = orc.heat_flux(p, parts, gp)
    scale = orc.heat_flux(p, dict(parts, w=np.abs(parts["w"])), np.abs(gp))  # magnitude of the terms
    assert abs(d["heat_flux"] - q_ref) <= 1e-9 * abs(scale) + 1e-300
    assert abs(d["field_energy"] - orc.field_energy(p, phi)) <= 1e-12 * orc.field_energy(p, phi)
    assert d["n_global"] == 12100
    assert abs(d["sum_w"] - parts["w"].sum()) <= 1e-12 * np.abs(parts["w"]).sum()
    # chi in gyro-Bohm units: (Q / N) / (R0/L_T / R0) * omega0^2
    assert abs(d["chi_gb"] - d["heat_flux"] / 12100 / (p.rlt / p.R0) * p.omega0 ** 2) <= 1e-12 * abs(d["chi_gb"])
    ctx.close()


def test_diag_zero_field_zero_flux(G):
    cfg = synth.config("T")
    parts = synth.load_particles(cfg, 2000, seed=42, w_amp=0.1)
    ctx = ctx_for(G, "T")
    ctx.set_particles(parts)
    ctx.set_grid(G.GRID_GRADPHI, np.zeros((3, ctx.get_info().mgrid, 3)))
    assert ctx.diag()["heat_flux"] == 0.0
    ctx.close()


def test_itg_growth_then_saturation(G):
    """Class-A grid, Cyclone parameters, micell 10: log(field energy) grows
    linearly (R^2 >= 0.98 over >= 200 steps) and then saturates (late growth
    rate < 10 % of the linear rate)."""
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
    import itg_run
    rows = itg_run.run("A", steps=700, every=10, micell=10, echo=False)
    res = itg_run.check(rows)
    assert res["ok"], res
    assert all(np.isfinite(r["field_energy"]) and np.isfinite(r["chi_gb"]) for r in rows)
    assert len({r["particle_count"] for r in rows}) == 1
