"""GPU edge cases against the oracle (same tolerances as test_gpu_parity):
empty and ragged marker counts, markers on every boundary of the domain
(r = a0, a1; theta = 0, 2pi^-; zeta on plane boundaries and 2pi^-), markers
whose gyro-points leave the tile window (the L2 fallback of the tiled
deposit), zero weights."""
import math

import numpy as np
import pytest

import synth
from test_gpu_parity import G, TOL, assert_particles_close, ctx_for, rel_err, _smooth_field  # noqa: F401

pytestmark = pytest.mark.gpu
TWO_PI = 2 * math.pi


def _subset(parts, idx):
    out = {k: np.ascontiguousarray(v[idx]) for k, v in parts.items()}
    out["id"] = np.arange(len(idx), dtype=np.uint64)
    return out


@pytest.fixture(scope="module")
def Tcfg(orc):
    cfg = synth.config("T")
    p = orc.make_params(cfg)
    return cfg, p, orc.geometry(p)


def test_empty_particle_set(G, orc, Tcfg):
    cfg, p, g = Tcfg
    parts = _subset(synth.load_particles(cfg, 10, seed=1), np.arange(0))
    ctx = ctx_for(G, "T")
    ctx.set_particles(parts)
    ctx.charge()
    assert not np.any(ctx.get_grid(G.GRID_CHARGE))
    ctx.set_grid(G.GRID_MARKER, np.ones(p.mpsi + 1))
    ctx.step(1)
    got = ctx.get_particles()
    assert len(got["id"]) == 0
    assert ctx.stats()["n_local"] == 0


@pytest.mark.parametrize("n", [1, 31, 33, 257, 8193])
def test_ragged_counts_charge_and_push(G, orc, Tcfg, n):
    """Counts that leave a ragged warp, CTA and tile tail."""
    cfg, p, g = Tcfg
    parts = synth.load_particles(cfg, n, seed=100 + n, w_amp=0.1)
    grids = []
    for mode in (0, 1):
        ctx = ctx_for(G, "T")
        ctx.set_charge_mode(mode)
        ctx.set_particles(parts)
        ctx.charge()
        grids.append(ctx.get_grid(G.GRID_CHARGE))
    assert np.array_equal(grids[0], grids[1])  # tiled == direct, bitwise
    ref = orc.charge_global(p, parts)
    assert rel_err(grids[0], ref) <= 1e-8
    gp = _smooth_field(orc, p, g)
    ctx = ctx_for(G, "T")
    ctx.set_particles(parts)
    ctx.set_grid(G.GRID_GRADPHI, gp)
    Xa = {k: parts[k].copy() for k in orc.ATTRS}
    Xb = {k: parts[k].copy() for k in orc.ATTRS}
    ctx.push(1)
    ctx.push(2)
    orc.push(p, 1, Xa, Xb, parts["mu"], gp)
    orc.push(p, 2, Xa, Xb, parts["mu"], gp)
    got = ctx.get_particles()
    assert_particles_close({**{k: got[k] for k in orc.ATTRS}, "id": got["id"]}, {**Xa, "id": parts["id"]})


def _boundary_markers(cfg, p, g):
    """Every combination of boundary radii, angles and plane positions."""
    dz = TWO_PI / p.mzetamax
    rs = [p.a0, np.nextafter(p.a0, 1.0), 0.5 * (p.a0 + p.a1), np.nextafter(p.a1, 0.0), p.a1]
    ths = [0.0, np.nextafter(TWO_PI, 0.0), math.pi]
    zs = [0.0, dz, np.nextafter(dz, 0.0), np.nextafter(TWO_PI, 0.0), 0.5 * dz]
    rows = [(0.5 * r * r, th, z) for r in rs for th in ths for z in zs]
    n = len(rows)
    a = np.array(rows)
    rng = np.random.default_rng(7)
    return {"psi": a[:, 0], "theta": a[:, 1], "zeta": a[:, 2], "rho": rng.normal(0, 1, n) / p.omega0,
            "w": rng.uniform(-0.1, 0.1, n), "mu": rng.exponential(1.0, n), "id": np.arange(n, dtype=np.uint64)}


def test_boundary_markers_charge_and_push(G, orc, Tcfg):
    cfg, p, g = Tcfg
    parts = _boundary_markers(cfg, p, g)
    ctx = ctx_for(G, "T")
    ctx.set_particles(parts)
    ctx.charge()
    got = ctx.get_grid(G.GRID_CHARGE)
    ref = orc.charge_global(p, parts)
    assert rel_err(got, ref) <= 1e-8
    # charge is conserved exactly in the fixed point (A-7 clamping keeps every point on the grid)
    assert abs(got.sum() - ref.sum()) <= 1e-9 * np.abs(parts["w"]).sum()
    gp = _smooth_field(orc, p, g)
    ctx.set_grid(G.GRID_GRADPHI, gp)
    Xa = {k: parts[k].copy() for k in orc.ATTRS}
    Xb = {k: parts[k].copy() for k in orc.ATTRS}
    ctx.push(1)
    ctx.push(2)
    orc.push(p, 1, Xa, Xb, parts["mu"], gp)
    orc.push(p, 2, Xa, Xb, parts["mu"], gp)
    got = ctx.get_particles()
    assert_particles_close({**{k: got[k] for k in orc.ATTRS}, "id": got["id"]}, {**Xa, "id": parts["id"]})
    assert np.all((got["theta"] >= 0) & (got["theta"] < TWO_PI))
    assert np.all((got["zeta"] >= 0) & (got["zeta"] < TWO_PI))
    r = np.sqrt(2 * got["psi"])
    assert np.all((r >= p.a0 - 1e-12) & (r <= p.a1 + 1e-12))


def test_window_overflow_goes_through_L2(G, orc):
    """Markers with gyroradii far beyond the tile window's 3 rho_th cut: their
    out-of-window contributions take the deferred L2 path; the tiled result
    still equals the direct deposit bitwise and the oracle."""
    cfg = synth.config("A")
    p = orc.make_params(cfg)
    parts = synth.load_particles(cfg, 200_000, seed=9)
    big = np.arange(0, 200_000, 50)
    parts["mu"][big] *= 400.0  # rho x 20
    grids = []
    for mode in (0, 1):
        ctx = ctx_for(G, "A")
        ctx.set_charge_mode(mode)
        ctx.set_particles(parts)
        ctx.charge()
        grids.append(ctx.get_grid(G.GRID_CHARGE))
        if mode == 0:
            assert ctx.stats()["charge_global_fallback"] > 0
    assert np.array_equal(grids[0], grids[1])
    assert rel_err(grids[0], orc.charge_global(p, parts)) <= 1e-8


def test_zero_weights_give_zero_charge(G, Tcfg):
    cfg, p, g = Tcfg
    parts = synth.load_particles(cfg, 5000, seed=3)
    parts["w"][:] = 0.0
    ctx = ctx_for(G, "T")
    ctx.set_particles(parts)
    ctx.charge()
    assert not np.any(ctx.get_grid(G.GRID_CHARGE))


def test_fp32_gather_field_with_fp64_state(G, orc, Tcfg):
    """field_f32 (experiment): the gather field stored in fp32 next to an fp64
    state.  Its rounding (2^-24 relative) moves the pushed state far less than
    the P-0 tolerance."""
    cfg, p, g = Tcfg
    parts = synth.load_particles(cfg, 12100, seed=5, w_amp=0.1)
    gp = _smooth_field(orc, p, g)
    ctx = ctx_for(G, "T", field_f32=1)
    ctx.set_particles(parts)
    ctx.set_grid(G.GRID_GRADPHI, gp)
    Xa = {k: parts[k].copy() for k in orc.ATTRS}
    Xb = {k: parts[k].copy() for k in orc.ATTRS}
    ctx.push(1)
    ctx.push(2)
    orc.push(p, 1, Xa, Xb, parts["mu"], gp)
    orc.push(p, 2, Xa, Xb, parts["mu"], gp)
    got = ctx.get_particles()
    assert_particles_close({**{k: got[k] for k in orc.ATTRS}, "id": got["id"]}, {**Xa, "id": parts["id"]})


# ------------------------------------------------------------------ ABI regressions (round-1 advisor findings)
def test_step_host_twice_matches_oracle(G, orc, Tcfg):
    """gtcp_step_host: upload, one step, download the owned state AND mu (a
    bin inside the step reorders them together), twice in a row; each call's
    result matches the oracle step of the previous call's output."""
    cfg, p, g = Tcfg
    parts = synth.load_particles(cfg, 12100, seed=7, w_amp=0.05)
    ctx = G.Context(G.gtcp_default_params("T", bin_every=1))
    ctx.set_particles(parts)
    nm = orc.marker_norm(p, parts)
    ctx.set_grid(G.GRID_MARKER, nm)
    keys = ("psi", "theta", "zeta", "rho", "w", "mu")
    host = [np.ascontiguousarray(parts[k]).copy() for k in keys]
    for call in range(2):
        state = {k: host[i].copy() for i, k in enumerate(keys)}
        orc.step_global(p, state, nm)
        n = ctx.step_host(host, 1)
        assert n == 12100
        # compare as multisets keyed by mu (mu is never written, unique per marker)
        o1, o2 = np.argsort(host[5]), np.argsort(state["mu"])
        assert np.array_equal(host[5][o1], state["mu"][o2])
        for i, k in enumerate(keys[:5]):
            if k in ("theta", "zeta"):
                d = (host[i][o1] - state[k][o2] + math.pi) % TWO_PI - math.pi
                assert np.max(np.abs(d)) / TWO_PI <= TOL, (call, k)
            else:
                assert rel_err(host[i][o1], state[k][o2]) <= TOL, (call, k)
    ctx.close()


def test_step_host_capacity_error(G, Tcfg):
    cfg, p, g = Tcfg
    parts = synth.load_particles(cfg, 1000, seed=8)
    ctx = G.Context(G.gtcp_default_params("T"))
    ctx.set_particles(parts)
    ctx.set_grid(G.GRID_MARKER, np.ones(p.mpsi + 1))
    host = [np.ascontiguousarray(parts[k]).copy() for k in ("psi", "theta", "zeta", "rho", "w", "mu")]
    import ctypes as C
    ptrs = (C.POINTER(C.c_double) * 6)(*[h.ctypes.data_as(C.POINTER(C.c_double)) for h in host])
    nout = C.c_int64()
    s = G.lib().gtcp_step_host(ctx._h, 1000, 999, ptrs, 1, C.byref(nout))  # cap < owned count
    assert s == 6 and nout.value == 1000  # GTCP_ECAPACITY, count reported
    ctx.close()


def test_sample_particles_ids_fp32(G, Tcfg):
    """precision 32 + track_ids: sampled ids are the 64-bit ids (not the fp32
    state's element size)."""
    cfg, p, g = Tcfg
    parts = synth.load_particles(cfg, 5000, seed=9)
    parts["id"] = (np.arange(5000, dtype=np.uint64) * np.uint64(2654435761) + np.uint64(1 << 40))
    ctx = G.Context(G.gtcp_default_params("T", precision=32, track_ids=1))
    ctx.set_particles(parts)
    full = ctx.get_particles(("psi",))
    idx = np.array([0, 17, 4999, 2500, 123])
    smp = ctx.sample_particles(idx, ("psi",))
    assert np.array_equal(smp["id"], full["id"][idx])
    assert set(full["id"].tolist()) == set(parts["id"].tolist())
    ctx.close()


def test_step_reports_nonfinite(G, Tcfg):
    """A non-finite weight makes gtcp_step return GTCP_ENONFINITE
    instead of stepping a corrupt state silently; the deposit skips it."""
    cfg, p, g = Tcfg
    parts = synth.load_particles(cfg, 2000, seed=10)
    ok = synth.load_particles(cfg, 2000, seed=10)
    parts["w"] = parts["w"].copy()
    parts["w"][5] = np.nan
    ctx = G.Context(G.gtcp_default_params("T"))
    ctx.set_particles(parts)
    ctx.charge()
    rho = ctx.get_grid(G.GRID_CHARGE)
    assert np.all(np.isfinite(rho))
    ok_sub = {k: np.delete(v, 5) for k, v in ok.items()}
    assert rel_err(rho, orc_charge := __import__("oracle").charge_global(
        __import__("oracle").make_params(cfg), ok_sub)) <= 1e-8
    ctx.set_grid(G.GRID_MARKER, np.ones(p.mpsi + 1))
    with pytest.raises(G.GtcpError) as e:
        ctx.step(1)
    assert e.value.status == 7  # GTCP_ENONFINITE
    ctx.close()


def test_push_loop_fission_matches_fused(G, orc, Tcfg):
    """Loop-fission ablation (gather loop writing gbar, then update
    loop) computes the same stage as the fused push."""
    cfg, p, g = Tcfg
    parts = synth.load_particles(cfg, 12100, seed=13, w_amp=0.1)
    gp = _smooth_field(orc, p, g)
    outs = []
    for mode in (0, 1):
        ctx = ctx_for(G, "T")
        ctx.set_push_mode(mode)
        ctx.set_particles(parts)
        ctx.set_grid(G.GRID_GRADPHI, gp)
        ctx.push(1)
        ctx.push(2)
        outs.append(ctx.get_particles())
        ctx.close()
    o1, o2 = np.argsort(outs[0]["id"]), np.argsort(outs[1]["id"])
    for k in ("psi", "theta", "zeta", "rho", "w"):
        assert rel_err(outs[1][k][o2], outs[0][k][o1]) <= 1e-14, k


@pytest.mark.parametrize("size,n", [("T", 12100), ("A", 300_000)])
def test_update_binning_charge_ablation_bitwise(G, orc, size, n):
    """charge mode 2 (the paper's update binning: points binned by
    their own cell, one thread per super-cell, twin shared-memory copies) gives
    the bitwise-identical fixed-point grid of the product deposit."""
    cfg = synth.config(size)
    parts = synth.load_particles(cfg, n, seed=17, w_amp=0.1)
    grids = []
    for mode in (0, 2):
        ctx = ctx_for(G, size)
        ctx.set_charge_mode(mode)
        ctx.set_particles(parts)
        ctx.charge()
        grids.append(ctx.get_grid(G.GRID_CHARGE))
        ctx.close()
    assert np.array_equal(grids[0], grids[1])


def test_fused_stage_pipeline_step_parity_T(G, orc):
    """SURVEY §8(f) #1 (gtcp_set_fused): the push of each RK2 stage deposits
    the next stage's charge in the same kernel; one full step against the
    oracle's step, three times along its trajectory (config T)."""
    cfg = synth.config("T")
    p = orc.make_params(cfg)
    state = synth.load_particles(cfg, 12100, seed=51, w_amp=0.1)
    nm = orc.marker_norm(p, state)
    for _ in range(3):
        ctx = ctx_for(G, "T")
        ctx.set_fused(True)
        ctx.set_particles(state)
        ctx.set_grid(G.GRID_MARKER, nm)
        ctx.step(1)
        got = ctx.get_particles()
        ctx.close()
        ref = {k: v.copy() for k, v in state.items()}
        orc.step_global(p, ref, nm)
        assert_particles_close(got, ref)
        state = ref


def test_fused_stage_pipeline_matches_unfused_A(G):
    """Class-A grid, 2 M markers, 4 steps in two gtcp_step calls (a bin after
    step 3; the charge deposited by the last push of the first call is used by
    the second): the fused pipeline (7 of the 8 charges deposited inside the
    preceding push) gives the unfused trajectory within the fixed-point
    rounding of the charge (its scale has one bit of headroom), and its charge
    phase really shrank."""
    cfg = synth.config("A")
    parts = synth.load_particles(cfg, 2_000_000, seed=52, w_amp=0.1)
    outs, charge_ms = [], []
    for fused in (False, True):
        ctx = ctx_for(G, "A")
        ctx.set_fused(fused)
        ctx.set_particles(parts)
        ctx.set_timing(True)
        ctx.timings_reset()
        ctx.step(2)
        ctx.step(2)
        charge_ms.append(ctx.timings()["charge_ms"])
        outs.append(ctx.get_particles())
        ctx.close()
    o0, o1 = np.argsort(outs[0]["id"]), np.argsort(outs[1]["id"])
    assert np.array_equal(outs[0]["id"][o0], outs[1]["id"][o1])
    for k in ("psi", "rho", "w"):
        assert rel_err(outs[1][k][o1], outs[0][k][o0]) <= 1e-9, k
    for k in ("theta", "zeta"):
        d = (outs[1][k][o1] - outs[0][k][o0] + math.pi) % TWO_PI - math.pi
        assert np.max(np.abs(d)) <= 1e-9, k
    assert charge_ms[1] < 0.5 * charge_ms[0], charge_ms


def test_fused_stage_pipeline_rejects_unsupported(G):
    ctx = G.Context(G.gtcp_default_params("T", precision=32))
    with pytest.raises(Exception):
        ctx.set_fused(True)
    ctx.set_fused(False)
    ctx.close()
