"""Statistics of the seeded marker loader (L-2/L-3)."""
import math

import numpy as np

import synth


def test_loader_statistics():
    cfg = synth.config("A")
    n = 400000
    s = synth.load_particles(cfg, n, seed=1)
    r = np.sqrt(2 * s["psi"])
    B = 1.0 / (1.0 + r / cfg["R0"] * np.cos(s["theta"]))
    vpar = s["rho"] * cfg["omega0"] * B
    assert abs(vpar.mean()) < 5e-3
    assert abs((vpar ** 2).mean() - 1.0) < 1e-2
    assert abs((s["mu"] * B).mean() - 1.0) < 1e-2  # <v_perp^2/2> = 1
    assert np.abs(s["w"]).max() <= cfg["w_init_amp"]
    assert r.min() >= cfg["a0"] and r.max() <= cfg["a1"]
    # chi^2 of the (r, theta) histogram against density ~ r * J
    nr, nt = 8, 8
    H, re, te = np.histogram2d(r, s["theta"], bins=[nr, nt], range=[[cfg["a0"], cfg["a1"]], [0, 2 * math.pi]])
    rr = np.linspace(cfg["a0"], cfg["a1"], 801)
    tt = np.linspace(0, 2 * math.pi, 801)
    R, TH = np.meshgrid(rr, tt, indexing="ij")
    dens = R * (1 + R / cfg["R0"] * np.cos(TH)) ** 2
    E = np.zeros((nr, nt))
    for a in range(nr):
        for b in range(nt):
            m = (R >= re[a]) & (R < re[a + 1]) & (TH >= te[b]) & (TH < te[b + 1])
            E[a, b] = dens[m].sum()
    E *= n / E.sum()
    chi2 = ((H - E) ** 2 / E).sum()
    assert chi2 < 2 * nr * nt, chi2


def test_loader_deterministic():
    cfg = synth.config("T")
    a = synth.load_particles(cfg, 1000, seed=5)
    b = synth.load_particles(cfg, 1000, seed=5)
    for k in a:
        assert np.array_equal(a[k], b[k])
