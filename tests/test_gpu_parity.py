"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same seeded inputs.  Tolerances (north_star, P-0 normwise per array):
fp64 grids and particle coordinates within 1e-6 of ||oracle||_inf; counts,
bin keys and shift destinations bit-exact.  Angles compared on the circle."""
import math

import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu
TOL = 1e-6
TWO_PI = 2 * math.pi


@pytest.fixture(scope="module")
def G():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    torch.cuda.set_device(0)
    import paper_1510_05546_b200 as g
    g.lib()
    return g


def ctx_for(G, size, n_parts=None, **over):
    p = G.gtcp_default_params(size, track_ids=1, **over)
    return G.Context(p)


def rel_err(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def circ(a, b):
    return (a - b + math.pi) % TWO_PI - math.pi


def assert_particles_close(got: dict, ref: dict, keys=("psi", "theta", "zeta", "rho", "w")):
    order_g = np.argsort(got["id"])
    order_r = np.argsort(ref["id"])
    assert np.array_equal(got["id"][order_g], ref["id"][order_r])
    for k in keys:
        a, b = got[k][order_g], ref[k][order_r]
        if k in ("theta", "zeta"):
            err = float(np.max(np.abs(circ(a, b)))) / TWO_PI
        else:
            err = rel_err(a, b)
        assert err <= TOL, (k, err)


@pytest.fixture(scope="module")
def T(orc):
    cfg = synth.config("T")
    p = orc.make_params(cfg)
    parts = synth.load_particles(cfg, 12100, seed=1)
    return cfg, p, orc.geometry(p), parts


# ------------------------------------------------------------------ charge
@pytest.mark.parametrize("mode", [0, 1])
def test_charge_parity_T(G, orc, T, mode):
    cfg, p, g, parts = T
    ctx = ctx_for(G, "T")
    ctx.set_charge_mode(mode)
    ctx.set_particles(parts)
    ctx.charge()
    got = ctx.get_grid(G.GRID_CHARGE)
    ref = orc.charge_global(p, parts)
    assert got.shape == ref.shape
    assert rel_err(got, ref) <= TOL
    assert rel_err(got, ref) <= 1e-8  # 31-bit fixed-point contributions: far inside TOL


def test_charge_tiled_equals_direct_bitwise(G, T):
    cfg, p, g, parts = T
    grids = []
    for mode in (0, 1, 0):
        ctx = ctx_for(G, "T")
        ctx.set_charge_mode(mode)
        ctx.set_particles(parts)
        ctx.charge()
        grids.append(ctx.get_grid(G.GRID_CHARGE))
    assert np.array_equal(grids[0], grids[1]) and np.array_equal(grids[0], grids[2])


def test_charge_parity_A_grid(G, orc):
    """A-size grid (32,449 nodes x 64 planes, the bench's launch configuration)
    with 2M markers: full element-wise parity."""
    cfg = synth.config("A")
    p = orc.make_params(cfg)
    parts = synth.load_particles(cfg, 2_000_000, seed=3)
    ctx = ctx_for(G, "A")
    ctx.set_particles(parts)
    ctx.charge()
    got = ctx.get_grid(G.GRID_CHARGE)
    ref = orc.charge_global(p, parts)
    assert rel_err(got, ref) <= 1e-8
    st = ctx.stats()
    assert st["plane_clamps"] == 0


def test_marker_norm_parity(G, orc, T):
    cfg, p, g, parts = T
    ctx = ctx_for(G, "T")
    ctx.set_particles(parts)
    assert rel_err(ctx.get_grid(G.GRID_MARKER), orc.marker_norm(p, parts)) <= 1e-8


# ------------------------------------------------------------------ grid kernels
def test_poisson_smooth_parity(G, orc, T):
    cfg, p, g, parts = T
    ctx = ctx_for(G, "T")
    ctx.set_particles(parts)
    charge = orc.charge_global(p, parts)
    nm = orc.marker_norm(p, parts)
    ctx.set_grid(G.GRID_CHARGE, charge)
    ctx.set_grid(G.GRID_MARKER, nm)
    ctx.poisson_smooth()
    got = ctx.get_grid(G.GRID_PHI)
    ref = orc.poisson_smooth(p, charge, nm)
    assert rel_err(got, ref) <= TOL


def test_field_parity(G, orc, T):
    cfg, p, g, parts = T
    rng = np.random.default_rng(0)
    phi = orc.smooth(p, rng.standard_normal((p.mzetamax + 1, g.mgrid)))
    ctx = ctx_for(G, "T")
    ctx.set_grid(G.GRID_PHI, phi)
    ctx.field()
    got = ctx.get_grid(G.GRID_GRADPHI)
    ref = orc.field(p, phi)
    assert rel_err(got, ref) <= TOL


# ------------------------------------------------------------------ push
def _smooth_field(orc, p, g):
    """Gradient field of an analytic potential on the nodes (oracle field)."""
    K = p.mzetamax
    phi = np.zeros((K + 1, g.mgrid))
    for k in range(K + 1):
        for i in range(p.mpsi + 1):
            r = p.a0 + i * (p.a1 - p.a0) / p.mpsi
            j = np.arange(g.mtheta[i] + 1)
            ze = k * TWO_PI / K
            th = j * TWO_PI / g.mtheta[i] + ze * g.qtinv[i]
            phi[k, g.igrid[i]:g.igrid[i] + g.mtheta[i] + 1] = 0.02 * np.sin(6 * r) * np.cos(3 * th - 2 * ze)
    return orc.field(p, phi)


@pytest.mark.parametrize("size,n", [("T", 12100), ("A", 300_000)])
def test_push_parity_two_stages(G, orc, size, n):
    cfg = synth.config(size)
    p = orc.make_params(cfg)
    g = orc.geometry(p)
    parts = synth.load_particles(cfg, n, seed=5, w_amp=0.1)
    gp = _smooth_field(orc, p, g)
    ctx = ctx_for(G, size)
    ctx.set_particles(parts)
    ctx.set_grid(G.GRID_GRADPHI, gp)
    Xa = {k: parts[k].copy() for k in orc.ATTRS}
    Xb = {k: parts[k].copy() for k in orc.ATTRS}
    ctx.push(1)
    orc.push(p, 1, Xa, Xb, parts["mu"], gp)
    got = ctx.get_particles()
    assert_particles_close({**{k: got[k] for k in orc.ATTRS}, "id": got["id"]}, {**Xb, "id": parts["id"]})
    # the saved state is the untouched X0
    assert_particles_close({"psi": got["psi0"], "theta": got["theta0"], "zeta": got["zeta0"], "rho": got["rho0"],
                            "w": got["w0"], "id": got["id"]}, {**Xa, "id": parts["id"]})
    ctx.push(2)
    orc.push(p, 2, Xa, Xb, parts["mu"], gp)
    got = ctx.get_particles()
    assert_particles_close({**{k: got[k] for k in orc.ATTRS}, "id": got["id"]}, {**Xa, "id": parts["id"]})
    order = np.argsort(got["id"])
    assert np.array_equal(got["mu"][order], parts["mu"])  # mu never written


def test_push_zero_field_keeps_w_bitwise(G, orc, T):
    cfg, p, g, parts = T
    ctx = ctx_for(G, "T")
    ctx.set_particles(parts)
    ctx.set_grid(G.GRID_GRADPHI, np.zeros((p.mzetamax + 1, g.mgrid, 3)))
    ctx.push(1)
    ctx.push(2)
    got = ctx.get_particles()
    order = np.argsort(got["id"])
    assert np.array_equal(got["w"][order], parts["w"])


# ------------------------------------------------------------------ bin
def test_bin_keys_sorted_and_permutation(G, orc, T):
    cfg, p, g, parts = T
    ctx = ctx_for(G, "T")
    ctx.set_particles(parts)  # bins
    got = ctx.get_particles()
    keys = orc.bin_key(p, got, nmu=G.gtcp_default_params("T").bin_mu)  # H-4 incl. mu sub-bins
    assert np.all(np.diff(keys) >= 0)
    order = np.argsort(got["id"])
    assert np.array_equal(got["id"][order], parts["id"])
    for k in ("psi", "theta", "zeta", "rho", "w", "mu"):
        assert np.array_equal(got[k][order], parts[k])  # bitwise: a permutation only


# ------------------------------------------------------------------ step
def test_step_parity_T_five_steps(G, orc, T):
    """reset both sides to the oracle state, run one full step
    (two RK stages of charge, poisson_smooth, field, push, shift), compare;
    five times along the oracle trajectory (config T, "5 steps")."""
    cfg, p, g, parts = T
    state = {k: v.copy() for k, v in parts.items()}
    nm = orc.marker_norm(p, state)
    for step in range(5):
        ctx = ctx_for(G, "T")
        ctx.set_particles(state)
        ctx.set_grid(G.GRID_MARKER, nm)
        ctx.step(1)
        got = ctx.get_particles()
        ref = {k: v.copy() for k, v in state.items()}
        orc.step_global(p, ref, nm)
        assert_particles_close(got, ref)
        state = ref


# ------------------------------------------------------------------ full size (A, 207M markers)
@pytest.fixture(scope="module")
def A_full(G):
    ctx = ctx_for(G, "A")
    ctx.load()
    yield ctx
    ctx.close()


def test_full_A_charge_conservation_and_determinism(G, orc, A_full):
    """Full class A (207,097,600 markers, P:522 x 64 planes) in the bench's
    launch configuration: deposited charge equals sum(w) (partition of unity),
    the smem-tiled kernel equals the direct-L2 kernel bitwise, reruns are
    bitwise identical (fixed-point accumulation)."""
    ctx = A_full
    info = ctx.get_info()
    assert info.n_local == 100 * (32449 - 90) * 64
    cfg = synth.config("A")
    g = orc.geometry(orc.make_params(cfg))
    ctx.charge()
    a = ctx.get_grid(G.GRID_CHARGE)
    st = ctx.stats()
    canon = sum(a[:64, g.igrid[i]:g.igrid[i] + g.mtheta[i]].sum() for i in range(cfg["mpsi"] + 1))
    assert abs(canon - st["sum_w"]) <= 1e-9 * info.n_local * cfg["w_init_amp"] / 2
    ctx.charge()
    b = ctx.get_grid(G.GRID_CHARGE)
    assert np.array_equal(a, b)
    ctx.set_charge_mode(1)
    ctx.charge()
    c = ctx.get_grid(G.GRID_CHARGE)
    ctx.set_charge_mode(0)
    assert np.array_equal(a, c)


def test_full_A_push_sampled(G, orc, A_full):
    """Full-size push: sampled particles before/after one stage-1 push match
    the oracle's push of those particles on the GPU's own field."""
    ctx = A_full
    cfg = synth.config("A")
    p = orc.make_params(cfg)
    ctx.charge()
    ctx.poisson_smooth()
    ctx.field()
    gp = ctx.get_grid(G.GRID_GRADPHI)
    n = ctx.get_info().n_local
    idx = np.sort(np.random.default_rng(0).choice(n, 20000, replace=False))
    before = ctx.sample_particles(idx)
    ctx.push(1)
    after = ctx.sample_particles(idx)
    Xa = {k: before[k].copy() for k in orc.ATTRS}
    Xb = {k: before[k].copy() for k in orc.ATTRS}
    orc.push(p, 1, Xa, Xb, before["mu"], gp)
    assert_particles_close({**{k: after[k] for k in orc.ATTRS}, "id": after["id"]}, {**Xb, "id": before["id"]})
    ctx.push(2)  # leave the context at a step boundary


def test_device_loader_statistics(G):
    ctx = ctx_for(G, "A", mzetamax=4)
    ctx.load()
    parts = ctx.get_particles(("psi", "theta", "zeta", "rho", "w", "mu"))
    cfg = synth.config("A")
    r = np.sqrt(2 * parts["psi"])
    B = 1.0 / (1.0 + r / cfg["R0"] * np.cos(parts["theta"]))
    vpar = parts["rho"] * cfg["omega0"] * B
    assert abs(vpar.mean()) < 5e-3
    assert abs((vpar ** 2).mean() - 1.0) < 1e-2
    assert abs((parts["mu"] * B).mean() - 1.0) < 1e-2
    assert r.min() >= cfg["a0"] and r.max() <= cfg["a1"]
    assert parts["zeta"].min() >= 0 and parts["zeta"].max() < 4 * TWO_PI / 4 + 1e-12


# ------------------------------------------------------------------ multi-GPU
def _ngpus():
    import torch
    return torch.cuda.device_count()


@pytest.mark.parametrize("args", [["--size", "T", "--mzetamax", "8"], ["--size", "A", "--nparts", "1000000"],
                                  ["--size", "A", "--nparts", "1000000", "--npartdom", "2"],
                                  ["--size", "A", "--nparts", "1000000", "--nradial", "2", "--precision", "32"]])
def test_toroidal_decomposition_parity_2gpu(G, args):
    """Decomposition over 2 GPUs against the oracle's single-domain step:
    toroidal (NCCL shift, ghost-plane charge merge, halo exchange), particle
    replicas (section charge allreduce, plane-split Poisson) and radial
    windows with the fp32 state (radial shift)."""
    import os
    import subprocess
    import sys
    if _ngpus() < 2:
        pytest.skip("needs 2 GPUs")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29533", os.path.join(root, "tests", "dist_parity.py")] + args
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert '"ok": true' in r.stdout


# ------------------------------------------------------------------ fp32 state (class D precision)
TOL32 = 1e-4


def _round32(parts):
    out = dict(parts)
    for k in ("psi", "theta", "zeta", "rho", "w", "mu"):
        out[k] = parts[k].astype(np.float32).astype(np.float64)
    # keep angles inside [0, 2 pi) after rounding
    for k in ("theta", "zeta"):
        out[k] = np.where(out[k] >= TWO_PI, 0.0, out[k])
    return out


def test_fp32_charge_and_step_parity(G, orc, T):
    """precision = 32: fp32 particle state, fp64 arithmetic.  Charge grid and
    one full step against the oracle fed the same fp32-rounded state."""
    cfg, p, g, parts = T
    parts32 = _round32(parts)
    ctx = G.Context(G.gtcp_default_params("T", track_ids=1, precision=32))
    ctx.set_particles(parts32)
    ctx.charge()
    got = ctx.get_grid(G.GRID_CHARGE)
    ref = orc.charge_global(p, parts32)
    assert rel_err(got, ref) <= TOL32
    nm = orc.marker_norm(p, parts32)
    ctx2 = G.Context(G.gtcp_default_params("T", track_ids=1, precision=32))
    ctx2.set_particles(parts32)
    ctx2.set_grid(G.GRID_MARKER, nm)
    ctx2.step(1)
    gotp = ctx2.get_particles()
    ref_state = {k: v.copy() for k, v in parts32.items()}
    orc.step_global(p, ref_state, nm)
    o1, o2 = np.argsort(gotp["id"]), np.argsort(ref_state["id"])
    assert np.array_equal(gotp["id"][o1], ref_state["id"][o2])
    for k in ("psi", "rho", "w"):
        assert rel_err(gotp[k][o1], ref_state[k][o2]) <= TOL32, k
    for k in ("theta", "zeta"):
        assert float(np.max(np.abs(circ(gotp[k][o1], ref_state[k][o2])))) / TWO_PI <= TOL32, k


def test_fp32_full_A_load_charge_conservation(G, orc):
    """fp32 store at full class A size: load, charge conservation, tiled == direct."""
    ctx = G.Context(G.gtcp_default_params("A", precision=32))
    ctx.load()
    ctx.charge()
    a = ctx.get_grid(G.GRID_CHARGE)
    st = ctx.stats()
    cfg = synth.config("A")
    g = orc.geometry(orc.make_params(cfg))
    canon = sum(a[:64, g.igrid[i]:g.igrid[i] + g.mtheta[i]].sum() for i in range(cfg["mpsi"] + 1))
    n = ctx.get_info().n_local
    assert abs(canon - st["sum_w"]) <= 1e-9 * n * cfg["w_init_amp"] / 2
    ctx.set_charge_mode(1)
    ctx.charge()
    assert np.array_equal(a, ctx.get_grid(G.GRID_CHARGE))
    ctx.step(2)
    assert ctx.stats()["n_global"] == n
    ctx.close()


def test_fp32_D_geometry_charge_and_push(G, orc):
    """Class D geometry (mpsi=768, mthetamax=5632: 2,406,883 nodes per plane),
    fp32 state, 4 planes to keep the oracle fast: charge and a stage-1 push
    against the oracle on the same fp32-rounded markers."""
    over = dict(mzetamax=4)
    cfg = synth.config("D", **over)
    p = orc.make_params(cfg)
    g = orc.geometry(p)
    assert g.mgrid == 2406883
    parts = _round32(synth.load_particles(cfg, 200_000, seed=4, w_amp=0.1))
    ctx = G.Context(G.gtcp_default_params("D", track_ids=1, precision=32, **over))
    ctx.set_particles(parts)
    ctx.charge()
    assert rel_err(ctx.get_grid(G.GRID_CHARGE), orc.charge_global(p, parts)) <= TOL32
    gp = _smooth_field(orc, p, g)
    ctx.set_grid(G.GRID_GRADPHI, gp)
    Xa = {k: parts[k].copy() for k in orc.ATTRS}
    Xb = {k: parts[k].copy() for k in orc.ATTRS}
    ctx.push(1)
    orc.push(p, 1, Xa, Xb, parts["mu"], gp)
    got = ctx.get_particles()
    o1, o2 = np.argsort(got["id"]), np.argsort(parts["id"])
    for k in ("psi", "rho", "w"):
        assert rel_err(got[k][o1], Xb[k][o2]) <= TOL32, k
    for k in ("theta", "zeta"):
        assert float(np.max(np.abs(circ(got[k][o1], Xb[k][o2])))) / TWO_PI <= TOL32, k
