"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This module holds configuration presets and the marker-loading recipe only --
none of the hot-path arithmetic (charge stencil, gather, push, shift).  Both
the oracle (``oracle/``) and the product library (``paper_1510_05546_b200``)
consume its outputs; neither is imported here.

Presets (BASELINE.json ``configs``; paper Tab.2 sizes for pins):
    T  mpsi=16  mthetamax=64   mzetamax=2  micell=10   (toy, oracle in seconds)
    A  mpsi=90  mthetamax=640  mzetamax=64 micell=100
    B  mpsi=192 mthetamax=1408 mzetamax=64 micell=100
    C  mpsi=384 mthetamax=2816 mzetamax=64 micell=100
    D  mpsi=768 mthetamax=5632 mzetamax=64 micell=100
    a..d: the paper's Tab.2 sizes 90/640, 180/1280, 360/2560, 720/5120.

Physics constants: Cyclone case, a/rho_i =
125*mpsi/90 (fig:convergence P:729 ladder), dt = 0.06, R0/a = 2.78.

Loading recipe (L-2, L-3): gyrocentre density uniform in
physical space, i.e. marker density in (r, theta) proportional to
r * J with J = (1 + (r/R0) cos theta)^2; zeta uniform; v_par ~ N(0,1)
and v_perp^2 = -2 ln U, each truncated at vcut = 5; mu = v_perp^2 / (2 B),
rho_par = v_par / (omega0 B) with the equilibrium B = 1/(1 + (r/R0) cos theta)
evaluated here as part of the recipe; w ~ U(-w_init_amp, w_init_amp).
Random numbers come from numpy's counter-based Philox keyed by the seed.
"""
from __future__ import annotations

import math

import numpy as np

SIZES = {
    "T": (16, 64, 2, 10),
    "A": (90, 640, 64, 100),
    "B": (192, 1408, 64, 100),
    "C": (384, 2816, 64, 100),
    "D": (768, 5632, 64, 100),
    "a": (90, 640, 64, 100),
    "b": (180, 1280, 64, 100),
    "c": (360, 2560, 64, 100),
    "d": (720, 5120, 64, 100),
}


def config(size: str = "T", **over) -> dict:
    """Full parameter dict for a preset (names follow the paper / C ABI)."""
    mpsi, mthetamax, mzetamax, micell = SIZES[size]
    cfg = dict(
        size=size, mpsi=mpsi, mthetamax=mthetamax, mzetamax=mzetamax, micell=micell,
        a0=0.1, a1=0.9, R0=2.78, omega0=125.0 * mpsi / 90.0,
        q0=0.854, q2=2.184, rln=2.2, rlt=6.9, tau=1.0, dt=0.06,
        paranl=1, drifts=1, poisson_iters=20, jacobi_omega=1.0,
        w_init_amp=1e-3, vcut=5.0,
    )
    cfg.update(over)
    return cfg


def load_particles(cfg: dict, n: int, seed: int, zeta_lo: float = 0.0,
                   zeta_hi: float = 2.0 * math.pi, w_amp: float | None = None) -> dict:
    """Draw ``n`` markers (L-2/L-3).  Returns SoA float64 arrays psi, theta,
    zeta, rho, w, mu and a uint64 ``id`` (0..n-1)."""
    rng = np.random.Generator(np.random.Philox(seed))
    a0, a1, R0 = cfg["a0"], cfg["a1"], cfg["R0"]
    vcut = cfg["vcut"]
    amp = cfg["w_init_amp"] if w_amp is None else w_amp
    jmax = (1.0 + a1 / R0) ** 2
    r = np.empty(0)
    th = np.empty(0)
    while r.size < n:
        m = max(1024, int(1.3 * (n - r.size)))
        rr = np.sqrt(a0 * a0 + (a1 * a1 - a0 * a0) * rng.random(m))
        tt = 2.0 * math.pi * rng.random(m)
        J = (1.0 + rr / R0 * np.cos(tt)) ** 2
        keep = rng.random(m) * jmax < J
        r = np.concatenate([r, rr[keep]])
        th = np.concatenate([th, tt[keep]])
    r = r[:n]
    th = th[:n]
    zeta = zeta_lo + (zeta_hi - zeta_lo) * rng.random(n)
    zeta = np.where(zeta >= zeta_hi, zeta_lo, zeta)

    def truncated(draw):
        v = draw(n)
        bad = np.abs(v) > vcut
        while bad.any():
            v[bad] = draw(int(bad.sum()))
            bad = np.abs(v) > vcut
        return v

    vpar = truncated(lambda m: rng.standard_normal(m))
    vperp = truncated(lambda m: np.sqrt(-2.0 * np.log1p(-rng.random(m))))
    B = 1.0 / (1.0 + r / R0 * np.cos(th))
    return dict(
        psi=0.5 * r * r,
        theta=th,
        zeta=zeta,
        rho=vpar / (cfg["omega0"] * B),
        w=amp * (2.0 * rng.random(n) - 1.0),
        mu=vperp * vperp / (2.0 * B),
        id=np.arange(n, dtype=np.uint64),
    )


def analytic_phi(cfg: dict, r, theta, zeta, amp: float = 1e-2):
    """A smooth prescribed potential for push tests (SURVEY §8(d) recipe):
    phi = amp * sin(6 r) * cos(3 theta - 2 zeta).  Returns phi and its
    partial derivatives (d/dr, d/dtheta, d/dzeta)."""
    s, c = np.sin(6 * r), np.cos(6 * r)
    arg = 3 * theta - 2 * zeta
    phi = amp * s * np.cos(arg)
    return phi, amp * 6 * c * np.cos(arg), -amp * 3 * s * np.sin(arg), amp * 2 * s * np.sin(arg)
