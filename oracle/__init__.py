"""CPU oracle of the GTC-P hot path (arXiv:1510.05546) -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import this package.  The product package
``paper_1510_05546_b200`` never imports it and shares no code with it.

This module is argument marshalling (ctypes + numpy) around ``gtcp_oracle.c``;
every step of the arithmetic lives in that C file, which cites the paper
passage (``P:n`` = PAPER.md line n) or SURVEY.md §8(c) reading it follows.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gtcp_oracle.c")
_SRC_OMP = os.path.join(_HERE, "gtcp_oracle_omp.c")
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (fp64, -ffp-contract=off: no fused a*b+c)."""
    os.makedirs(os.path.dirname(_LIB_PATH), exist_ok=True)
    if force or not os.path.exists(_LIB_PATH) or \
            os.path.getmtime(_LIB_PATH) < max(os.path.getmtime(_SRC), os.path.getmtime(_SRC_OMP)):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
                               "-fPIC", "-shared", "-o", tmp, _SRC, _SRC_OMP, "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


class Params(C.Structure):
    _fields_ = [
        ("mpsi", C.c_int32), ("mthetamax", C.c_int32), ("mzetamax", C.c_int32),
        ("paranl", C.c_int32), ("drifts", C.c_int32), ("poisson_iters", C.c_int32),
        ("a0", C.c_double), ("a1", C.c_double), ("R0", C.c_double), ("omega0", C.c_double),
        ("q0", C.c_double), ("q2", C.c_double), ("rln", C.c_double), ("rlt", C.c_double),
        ("tau", C.c_double), ("dt", C.c_double), ("jacobi_omega", C.c_double),
    ]


def make_params(cfg: dict, **over) -> Params:
    """Build oracle parameters from a config dict (``synth.config``)."""
    d = dict(cfg)
    d.update(over)
    p = Params()
    for name, _ in Params._fields_:
        setattr(p, name, d[name])
    return p


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        P = C.POINTER(Params)
        d = C.POINTER(C.c_double)
        i32 = C.POINTER(C.c_int32)
        i64 = C.POINTER(C.c_int64)
        sig = {
            "orc_geometry": (C.c_int64, [P, i32, i64, i32, d]),
            "orc_prof": (C.c_double, [C.c_double]),
            "orc_qprofile": (C.c_double, [P, C.c_double]),
            "orc_bfield": (C.c_double, [P, C.c_double, C.c_double]),
            "orc_deposit": (C.c_int64, [P, C.c_int64, d, d, d, d, d, C.c_int32, C.c_int32, d]),
            "orc_charge_reduce_global": (None, [P, d]),
            "orc_marker_norm": (None, [P, C.c_int64, d, d, d, d, d]),
            "orc_smooth": (None, [P, d]),
            "orc_zonal_solve": (None, [P, d, d]),
            "orc_poisson_smooth": (None, [P, d, d, d]),
            "orc_jacobi_plane": (None, [P, C.c_int32, d, d]),
            "orc_gyro_op": (None, [P, C.c_int32, d, d]),
            "orc_field": (None, [P, d, d]),
            "orc_gather": (None, [P, C.c_int64, d, d, d, d, C.c_int32, C.c_int32, d, d]),
            "orc_rhs": (None, [P, d, C.c_double, d, d]),
            "orc_push": (C.c_int64, [P, C.c_int32, C.c_int64, C.POINTER(d), C.POINTER(d), d,
                                     C.c_int32, C.c_int32, d]),
            "orc_shift_dest": (None, [P, C.c_int64, d, C.c_int32, i32]),
            "orc_bin_key": (None, [P, C.c_int64, d, d, d, d, C.c_int32, C.c_int32, C.c_int32, i64]),
            "orc_heat_flux": (C.c_double, [P, C.c_int64, d, d, d, d, d, d, C.c_int32, C.c_int32, d]),
            "orc_omp_threads": (C.c_int, []),
            "orc_deposit_replicas": (C.c_int64, [P, C.c_int64, d, d, d, d, d, C.c_int32, C.c_int32, d, C.c_int64]),
            "orc_push_omp": (C.c_int64, [P, C.c_int32, C.c_int64, C.POINTER(d), C.POINTER(d), d,
                                         C.c_int32, C.c_int32, d]),
            "orc_shift_dest_omp": (None, [P, C.c_int64, d, C.c_int32, i32]),
            "orc_radial_windows": (None, [P, C.c_int32, i32]),
            "orc_radial_dest": (None, [P, C.c_int64, d, C.c_int32, i32, i32]),
        }
        for name, (res, args) in sig.items():
            f = getattr(_lib, name)
            f.restype = res
            f.argtypes = args
    return _lib


def _d(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


@dataclass
class Geometry:
    mtheta: np.ndarray
    igrid: np.ndarray
    itran: np.ndarray
    qtinv: np.ndarray
    mgrid: int


def geometry(p: Params) -> Geometry:
    n = p.mpsi + 1
    mtheta = np.zeros(n, np.int32)
    igrid = np.zeros(n + 1, np.int64)
    itran = np.zeros(n, np.int32)
    qtinv = np.zeros(n, np.float64)
    mgrid = lib().orc_geometry(C.byref(p), mtheta.ctypes.data_as(C.POINTER(C.c_int32)),
                               igrid.ctypes.data_as(C.POINTER(C.c_int64)),
                               itran.ctypes.data_as(C.POINTER(C.c_int32)), _d(qtinv))
    return Geometry(mtheta, igrid, itran, qtinv, int(mgrid))


def prof(r: float) -> float:
    return lib().orc_prof(r)


def qprofile(p: Params, r: float) -> float:
    return lib().orc_qprofile(C.byref(p), r)


def bfield(p: Params, r: float, theta: float) -> float:
    return lib().orc_bfield(C.byref(p), r, theta)


def deposit(p: Params, parts: dict, k0: int = 0, P: int | None = None, w=None):
    """Charge deposit (Q-1..Q-6) onto P+1 local planes; returns (grid, nclamp)."""
    g = geometry(p)
    P = p.mzetamax if P is None else P
    grid = np.zeros((P + 1) * g.mgrid)
    a = [_f64(parts[k]) for k in ("psi", "theta", "zeta", "mu")]
    ww = _f64(parts["w"] if w is None else w)
    nclamp = lib().orc_deposit(C.byref(p), len(ww), *[_d(x) for x in a], _d(ww), k0, P, _d(grid))
    return grid.reshape(P + 1, g.mgrid), nclamp


def charge_reduce_global(p: Params, grid: np.ndarray) -> np.ndarray:
    out = _f64(grid).copy()
    lib().orc_charge_reduce_global(C.byref(p), _d(out))
    return out


def charge_global(p: Params, parts: dict) -> np.ndarray:
    """Deposit + Q-7 reductions on the single-domain (global) grid."""
    grid, _ = deposit(p, parts)
    return charge_reduce_global(p, grid)


def marker_norm(p: Params, parts: dict) -> np.ndarray:
    nm = np.zeros(p.mpsi + 1)
    a = [_f64(parts[k]) for k in ("psi", "theta", "zeta", "mu")]
    lib().orc_marker_norm(C.byref(p), len(a[0]), *[_d(x) for x in a], _d(nm))
    return nm


def smooth(p: Params, f: np.ndarray) -> np.ndarray:
    out = _f64(f).copy()
    lib().orc_smooth(C.byref(p), _d(out))
    return out


def zonal_solve(p: Params, nbar: np.ndarray) -> np.ndarray:
    out = np.zeros(p.mpsi + 1)
    lib().orc_zonal_solve(C.byref(p), _d(_f64(nbar)), _d(out))
    return out


def poisson_smooth(p: Params, charge: np.ndarray, nm: np.ndarray) -> np.ndarray:
    charge = _f64(charge)
    phi = np.zeros_like(charge)
    lib().orc_poisson_smooth(C.byref(p), _d(charge), _d(_f64(nm)), _d(phi))
    return phi


def jacobi_plane(p: Params, k: int, rhs: np.ndarray) -> np.ndarray:
    out = np.zeros_like(_f64(rhs))
    lib().orc_jacobi_plane(C.byref(p), k, _d(_f64(rhs)), _d(out))
    return out


def gyro_op(p: Params, k: int, f: np.ndarray) -> np.ndarray:
    out = np.zeros_like(_f64(f))
    lib().orc_gyro_op(C.byref(p), k, _d(_f64(f)), _d(out))
    return out


def field(p: Params, phi: np.ndarray) -> np.ndarray:
    phi = _f64(phi)
    out = np.zeros(phi.size * 3)
    lib().orc_field(C.byref(p), _d(phi), _d(out))
    return out.reshape(phi.shape + (3,))


def gather(p: Params, parts: dict, gradphi: np.ndarray, k0: int = 0, P: int | None = None):
    P = p.mzetamax if P is None else P
    a = [_f64(parts[k]) for k in ("psi", "theta", "zeta", "mu")]
    out = np.zeros((len(a[0]), 3))
    lib().orc_gather(C.byref(p), len(a[0]), *[_d(x) for x in a], k0, P, _d(_f64(gradphi).ravel()), _d(out))
    return out


def rhs(p: Params, X, mu: float, gbar) -> np.ndarray:
    x = _f64(X)
    gb = _f64(gbar)
    out = np.zeros(5)
    lib().orc_rhs(C.byref(p), _d(x), float(mu), _d(gb), _d(out))
    return out


ATTRS = ("psi", "theta", "zeta", "rho", "w")


def push(p: Params, stage: int, Xa: dict, Xb: dict, mu, gradphi, k0: int = 0, P: int | None = None) -> int:
    """One RK2 stage in place (U-7): stage 1 writes Xb, stage 2 writes Xa."""
    P = p.mzetamax if P is None else P
    for dct in (Xa, Xb):
        for k in ATTRS:
            dct[k] = _f64(dct[k])
    pa = (C.POINTER(C.c_double) * 5)(*[_d(Xa[k]) for k in ATTRS])
    pb = (C.POINTER(C.c_double) * 5)(*[_d(Xb[k]) for k in ATTRS])
    mu = _f64(mu)
    return lib().orc_push(C.byref(p), stage, len(mu), pa, pb, _d(mu), k0, P, _d(_f64(gradphi).ravel()))


def shift_dest(p: Params, zeta: np.ndarray, P: int) -> np.ndarray:
    z = _f64(zeta)
    out = np.zeros(len(z), np.int32)
    lib().orc_shift_dest(C.byref(p), len(z), _d(z), P, out.ctypes.data_as(C.POINTER(C.c_int32)))
    return out


def heat_flux(p: Params, parts: dict, gradphi: np.ndarray, k0: int = 0, P: int | None = None) -> float:
    """Diagnostic heat flux sum_p w E_kin v_E,r with the gathered field."""
    P = p.mzetamax if P is None else P
    a = [_f64(parts[k]) for k in ("psi", "theta", "zeta", "rho", "w", "mu")]
    return float(lib().orc_heat_flux(C.byref(p), len(a[0]), *[_d(x) for x in a], k0, P,
                                     _d(_f64(gradphi).ravel())))


def field_energy(p: Params, phi: np.ndarray) -> float:
    """Sum of phi^2 over the canonical nodes (j < mtheta) of planes 0..mzetamax-1."""
    g = geometry(p)
    phi = _f64(phi).reshape(-1, g.mgrid)
    s = 0.0
    for i in range(p.mpsi + 1):
        s += float(np.sum(phi[:p.mzetamax, g.igrid[i]:g.igrid[i] + g.mtheta[i]] ** 2))
    return s


def omp_threads() -> int:
    return int(lib().orc_omp_threads())


def deposit_replicas(p: Params, parts: dict, k0: int = 0, P: int | None = None):
    """orc_deposit over all OpenMP threads with per-thread grid replicas summed
    in thread order; same result as deposit() up to summation order."""
    g = geometry(p)
    P = p.mzetamax if P is None else P
    grid = np.zeros((P + 1) * g.mgrid)
    a = [_f64(parts[k]) for k in ("psi", "theta", "zeta", "mu", "w")]
    nclamp = lib().orc_deposit_replicas(C.byref(p), len(a[0]), *[_d(x) for x in a], k0, P, _d(grid), grid.size)
    return grid.reshape(P + 1, g.mgrid), nclamp


def push_omp(p: Params, stage: int, Xa: dict, Xb: dict, mu, gradphi, k0: int = 0, P: int | None = None) -> int:
    """push() split over all OpenMP threads by particle range."""
    P = p.mzetamax if P is None else P
    for dct in (Xa, Xb):
        for k in ATTRS:
            dct[k] = _f64(dct[k])
    pa = (C.POINTER(C.c_double) * 5)(*[_d(Xa[k]) for k in ATTRS])
    pb = (C.POINTER(C.c_double) * 5)(*[_d(Xb[k]) for k in ATTRS])
    mu = _f64(mu)
    return lib().orc_push_omp(C.byref(p), stage, len(mu), pa, pb, _d(mu), k0, P, _d(_f64(gradphi).ravel()))


def shift_dest_omp(p: Params, zeta: np.ndarray, P: int) -> np.ndarray:
    z = _f64(zeta)
    out = np.zeros(len(z), np.int32)
    lib().orc_shift_dest_omp(C.byref(p), len(z), _d(z), P, out.ctypes.data_as(C.POINTER(C.c_int32)))
    return out


def radial_windows(p: Params, K: int) -> np.ndarray:
    """G-6 equal-area radial windows snapped to rings: ring indices bound[0..K]."""
    out = np.zeros(K + 1, np.int32)
    lib().orc_radial_windows(C.byref(p), K, out.ctypes.data_as(C.POINTER(C.c_int32)))
    return out


def radial_dest(p: Params, psi: np.ndarray, K: int) -> np.ndarray:
    """H-2 radial owner window of each particle (G-6 windows)."""
    b = radial_windows(p, K)
    z = _f64(psi)
    out = np.zeros(len(z), np.int32)
    lib().orc_radial_dest(C.byref(p), len(z), _d(z), K, b.ctypes.data_as(C.POINTER(C.c_int32)),
                          out.ctypes.data_as(C.POINTER(C.c_int32)))
    return out


def bin_key(p: Params, parts: dict, k0: int = 0, P: int | None = None, nmu: int = 1) -> np.ndarray:
    """H-4 bin key; nmu > 1 refines it by magnetic-moment quantile sub-bins."""
    P = p.mzetamax if P is None else P
    a = [_f64(parts[k]) for k in ("psi", "theta", "zeta")]
    mu = _f64(parts["mu"]) if nmu > 1 else np.zeros(len(a[0]))
    out = np.zeros(len(a[0]), np.int64)
    lib().orc_bin_key(C.byref(p), len(a[0]), *[_d(x) for x in a], _d(mu), k0, P, nmu,
                      out.ctypes.data_as(C.POINTER(C.c_int64)))
    return out


def step_global(p: Params, parts: dict, nm: np.ndarray):
    """One full step on one domain (S-0 reading): for stage in (1, 2):
    charge -> poisson_smooth -> field -> push(stage).  (At one domain the shift
    moves nobody.)  ``parts`` is updated in place; returns per-stage grids."""
    Xa = {k: _f64(parts[k]).copy() for k in ATTRS}
    Xb = {k: v.copy() for k, v in Xa.items()}
    mu = _f64(parts["mu"])
    out = []
    for stage in (1, 2):
        src = Xa if stage == 1 else Xb
        cur = dict(src, mu=mu)
        ch = charge_global(p, cur)
        phi = poisson_smooth(p, ch, nm)
        gp = field(p, phi)
        push(p, stage, Xa, Xb, mu, gp)
        out.append((ch, phi, gp))
    for k in ATTRS:
        parts[k] = Xa[k]
    return out
