"""B200-native GTC-P hot path (arXiv:1510.05546): thin Python binding over libgtcp.so.

Argument marshalling only: every step of the hot path (charge, reductions,
poisson/smooth/field, gather+push, shift, bin) runs in the library's CUDA
kernels for sm_100a.  The names mirror the C ABI in ``include/gtcp.h``
(``gtcp_init`` -> ``Context(...)``, ``gtcp_charge`` -> ``Context.charge`` and
the module-level ``gtcp_*`` functions).  There is no CPU fallback: if the
library is missing or no GPU is present the calls raise.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GTCP_LIB_PATH") or os.path.join(_HERE, "_lib", "libgtcp.so")

ATTRS = ("psi", "theta", "zeta", "rho", "w", "mu", "psi0", "theta0", "zeta0", "rho0", "w0")
GRID_CHARGE, GRID_PHI, GRID_GRADPHI, GRID_MARKER = 0, 1, 2, 3
PHASES = ("charge", "charge_red", "poisson", "field", "push", "shift", "bin")
STATUS = {0: "OK", 1: "EINVAL", 2: "EINVARIANT", 3: "ENOMEM", 4: "ECUDA", 5: "ENCCL", 6: "ECAPACITY",
          7: "ENONFINITE", 8: "ESTATE"}


class GtcpError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"gtcp {STATUS.get(status, status)}: {msg}")
        self.status = status


class Params(C.Structure):
    _fields_ = [
        ("mpsi", C.c_int32), ("mthetamax", C.c_int32), ("mzetamax", C.c_int32), ("micell", C.c_int32),
        ("ntoroidal", C.c_int32), ("npartdom", C.c_int32), ("nradial", C.c_int32), ("bin_mu", C.c_int32),
        ("precision", C.c_int32), ("bin_every", C.c_int32),
        ("poisson_iters", C.c_int32), ("paranl", C.c_int32), ("drifts", C.c_int32), ("track_ids", C.c_int32),
        ("a0", C.c_double), ("a1", C.c_double), ("R0", C.c_double), ("omega0", C.c_double),
        ("q0", C.c_double), ("q2", C.c_double), ("rln", C.c_double), ("rlt", C.c_double),
        ("tau", C.c_double), ("dt", C.c_double), ("jacobi_omega", C.c_double), ("w_init_amp", C.c_double),
        ("vcut", C.c_double), ("capacity_factor", C.c_double), ("seed", C.c_uint64), ("field_f32", C.c_int32), ("reserved2", C.c_int32),
    ]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class Info(C.Structure):
    _fields_ = [("mgrid", C.c_int64), ("P", C.c_int32), ("k0", C.c_int32), ("rank_toroidal", C.c_int32),
                ("rank_particle", C.c_int32), ("rank_radial", C.c_int32), ("ring_lo", C.c_int32),
                ("ring_hi", C.c_int32), ("reserved1", C.c_int32), ("n_local", C.c_int64), ("capacity", C.c_int64),
                ("stage_next", C.c_int32), ("steps_done", C.c_int32)]


class Stats(C.Structure):
    _fields_ = [("n_local", C.c_int64), ("n_global", C.c_int64), ("sum_w", C.c_double), ("max_abs_w", C.c_double),
                ("movers_sent", C.c_int64), ("movers_recv", C.c_int64), ("reflections", C.c_int64),
                ("plane_clamps", C.c_int64), ("charge_global_fallback", C.c_int64), ("fx_shift", C.c_int32)]


class Diag(C.Structure):
    _fields_ = [("field_energy", C.c_double), ("heat_flux", C.c_double), ("chi_gb", C.c_double),
                ("sum_w", C.c_double), ("n_global", C.c_int64)]


class Timings(C.Structure):
    _fields_ = [("ms", C.c_double * 7), ("calls", C.c_int64 * 7), ("launches", C.c_int64),
                ("comm_bytes", C.c_int64 * 7)]


# every symbol declared in include/gtcp.h
SYMBOLS = ("gtcp_default_params", "gtcp_geometry", "gtcp_nccl_unique_id", "gtcp_init", "gtcp_destroy",
           "gtcp_strerror", "gtcp_info", "gtcp_load", "gtcp_set_particles", "gtcp_get_particles", "gtcp_charge",
           "gtcp_poisson_smooth", "gtcp_field", "gtcp_push", "gtcp_shift", "gtcp_bin", "gtcp_step",
           "gtcp_step_host", "gtcp_get_grid", "gtcp_set_grid", "gtcp_stats", "gtcp_timings", "gtcp_timings_reset",
           "gtcp_set_timing", "gtcp_set_charge_mode", "gtcp_sample_particles", "gtcp_loopback_create",
           "gtcp_loopback_destroy", "gtcp_init_loopback", "gtcp_diag", "gtcp_set_push_mode", "gtcp_set_fused")

_lib = None


def lib():
    """Load libgtcp.so (built by ``__graft_entry__.build()``); raise if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(LIB_PATH)
        vp, st = C.c_void_p, C.c_int
        dpp = C.POINTER(C.POINTER(C.c_double))
        sig = {
            "gtcp_default_params": (st, [C.c_char, C.POINTER(Params)]),
            "gtcp_geometry": (st, [C.POINTER(Params), C.POINTER(C.c_int32), C.POINTER(C.c_int64),
                                   C.POINTER(C.c_int32), C.POINTER(C.c_double), C.POINTER(C.c_int64)]),
            "gtcp_nccl_unique_id": (st, [vp]),
            "gtcp_init": (st, [C.POINTER(Params), C.c_int, C.c_int, vp, vp, C.POINTER(vp)]),
            "gtcp_destroy": (None, [vp]),
            "gtcp_strerror": (C.c_char_p, [vp]),
            "gtcp_info": (st, [vp, C.POINTER(Info)]),
            "gtcp_load": (st, [vp]),
            "gtcp_set_particles": (st, [vp, C.c_int64, dpp, C.POINTER(C.c_uint64)]),
            "gtcp_get_particles": (st, [vp, C.c_int64, C.POINTER(C.c_int64), dpp, C.POINTER(C.c_uint64)]),
            "gtcp_sample_particles": (st, [vp, C.c_int64, C.POINTER(C.c_int64), dpp, C.POINTER(C.c_uint64)]),
            "gtcp_charge": (st, [vp]),
            "gtcp_poisson_smooth": (st, [vp]),
            "gtcp_field": (st, [vp]),
            "gtcp_push": (st, [vp, C.c_int]),
            "gtcp_shift": (st, [vp]),
            "gtcp_bin": (st, [vp]),
            "gtcp_step": (st, [vp, C.c_int]),
            "gtcp_step_host": (st, [vp, C.c_int64, C.c_int64, dpp, C.c_int, C.POINTER(C.c_int64)]),
            "gtcp_loopback_create": (st, [C.c_int, C.POINTER(vp)]),
            "gtcp_loopback_destroy": (None, [vp]),
            "gtcp_init_loopback": (st, [C.POINTER(Params), C.c_int, C.c_int, vp, vp, C.POINTER(vp)]),
            "gtcp_get_grid": (st, [vp, C.c_int, C.c_int64, C.POINTER(C.c_double)]),
            "gtcp_set_grid": (st, [vp, C.c_int, C.c_int64, C.POINTER(C.c_double)]),
            "gtcp_stats": (st, [vp, C.POINTER(Stats)]),
            "gtcp_diag": (st, [vp, C.POINTER(Diag)]),
            "gtcp_timings": (st, [vp, C.POINTER(Timings)]),
            "gtcp_timings_reset": (st, [vp]),
            "gtcp_set_timing": (st, [vp, C.c_int]),
            "gtcp_set_charge_mode": (st, [vp, C.c_int]),
            "gtcp_set_push_mode": (st, [vp, C.c_int]),
            "gtcp_set_fused": (st, [vp, C.c_int]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _dp(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(C.POINTER(C.c_double))


def gtcp_default_params(size: str = "A", **over) -> Params:
    p = Params()
    s = lib().gtcp_default_params(size.encode(), C.byref(p))
    if s:
        raise GtcpError(s, f"unknown size {size!r}")
    for k, v in over.items():
        setattr(p, k, v)
    return p


def gtcp_geometry(p: Params) -> dict:
    n = p.mpsi + 1
    mtheta = np.zeros(n, np.int32)
    igrid = np.zeros(n + 1, np.int64)
    itran = np.zeros(n, np.int32)
    qtinv = np.zeros(n)
    mgrid = C.c_int64()
    s = lib().gtcp_geometry(C.byref(p), mtheta.ctypes.data_as(C.POINTER(C.c_int32)),
                            igrid.ctypes.data_as(C.POINTER(C.c_int64)), itran.ctypes.data_as(C.POINTER(C.c_int32)),
                            _dp(qtinv), C.byref(mgrid))
    if s:
        raise GtcpError(s, "geometry")
    return dict(mtheta=mtheta, igrid=igrid, itran=itran, qtinv=qtinv, mgrid=int(mgrid.value))


def gtcp_nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    s = lib().gtcp_nccl_unique_id(buf)
    if s:
        raise GtcpError(s, "ncclGetUniqueId")
    return buf.raw


class Context:
    """One rank's GTC-P hot-path state on the current CUDA device (gtcp_init)."""

    def __init__(self, params: Params, rank: int = 0, nranks: int = 1, nccl_id: bytes | None = None,
                 stream: int | None = None, loopback: "LoopbackHub | None" = None):
        self.params = params
        self._h = C.c_void_p()
        if loopback is not None:
            s = lib().gtcp_init_loopback(C.byref(params), rank, nranks, loopback.handle, C.c_void_p(stream or 0),
                                         C.byref(self._h))
        else:
            idbuf = C.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
            s = lib().gtcp_init(C.byref(params), rank, nranks, idbuf, C.c_void_p(stream or 0), C.byref(self._h))
        if s:
            msg = lib().gtcp_strerror(self._h).decode() if self._h.value else ""
            if self._h.value:
                lib().gtcp_destroy(self._h)
            self._h = C.c_void_p()
            raise GtcpError(s, f"init: {msg}")
        self.info = self.get_info()

    # -- helpers
    def _chk(self, s: int, what: str):
        if s:
            raise GtcpError(s, f"{what}: {lib().gtcp_strerror(self._h).decode()}")

    def close(self):
        if self._h and self._h.value:
            lib().gtcp_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def get_info(self) -> Info:
        i = Info()
        self._chk(lib().gtcp_info(self._h, C.byref(i)), "info")
        return i

    # -- particles
    def load(self):
        self._chk(lib().gtcp_load(self._h), "load")

    def set_particles(self, parts: dict):
        arrs = [np.ascontiguousarray(parts[k], dtype=np.float64) for k in ATTRS[:6]]
        n = len(arrs[0])
        ptrs = (C.POINTER(C.c_double) * 6)(*[_dp(a) for a in arrs])
        ids = parts.get("id")
        idp = None
        if ids is not None:
            ids = np.ascontiguousarray(ids, dtype=np.uint64)
            idp = ids.ctypes.data_as(C.POINTER(C.c_uint64))
        self._chk(lib().gtcp_set_particles(self._h, n, ptrs, idp), "set_particles")

    def get_particles(self, attrs=ATTRS) -> dict:
        n = self.get_info().n_local
        out = {k: np.empty(n) for k in attrs}
        ptrs = (C.POINTER(C.c_double) * 11)(*[(_dp(out[k]) if k in out else C.POINTER(C.c_double)()) for k in ATTRS])
        ids = np.empty(n, np.uint64) if self.params.track_ids else None
        nn = C.c_int64()
        self._chk(lib().gtcp_get_particles(self._h, n, C.byref(nn), ptrs,
                                           ids.ctypes.data_as(C.POINTER(C.c_uint64)) if ids is not None else None),
                  "get_particles")
        if ids is not None:
            out["id"] = ids
        return out

    def sample_particles(self, idx, attrs=ATTRS) -> dict:
        idx = np.ascontiguousarray(idx, dtype=np.int64)
        m = len(idx)
        out = {k: np.empty(m) for k in attrs}
        ptrs = (C.POINTER(C.c_double) * 11)(*[(_dp(out[k]) if k in out else C.POINTER(C.c_double)()) for k in ATTRS])
        ids = np.empty(m, np.uint64) if self.params.track_ids else None
        self._chk(lib().gtcp_sample_particles(self._h, m, idx.ctypes.data_as(C.POINTER(C.c_int64)), ptrs,
                                              ids.ctypes.data_as(C.POINTER(C.c_uint64)) if ids is not None else None),
                  "sample_particles")
        if ids is not None:
            out["id"] = ids
        return out

    # -- hot path
    def charge(self):
        self._chk(lib().gtcp_charge(self._h), "charge")

    def poisson_smooth(self):
        self._chk(lib().gtcp_poisson_smooth(self._h), "poisson_smooth")

    def field(self):
        self._chk(lib().gtcp_field(self._h), "field")

    def push(self, stage: int):
        self._chk(lib().gtcp_push(self._h, stage), "push")

    def shift(self):
        self._chk(lib().gtcp_shift(self._h), "shift")

    def bin(self):
        self._chk(lib().gtcp_bin(self._h), "bin")

    def step(self, nsteps: int = 1):
        self._chk(lib().gtcp_step(self._h, nsteps), "step")

    def step_host(self, arrays: list, nsteps: int = 1, n: int | None = None) -> int:
        """arrays: 6 pinned/contiguous fp64 host arrays (psi, theta, zeta, rho, w, mu) of equal capacity;
        the first n (default: all) are uploaded, the owned particles after the steps (live state and mu)
        are written back in place.  Returns the owned count."""
        cap = len(arrays[0])
        n = cap if n is None else n
        ptrs = (C.POINTER(C.c_double) * 6)(*[_dp(a) for a in arrays])
        nout = C.c_int64()
        self._chk(lib().gtcp_step_host(self._h, n, cap, ptrs, nsteps, C.byref(nout)), "step_host")
        return int(nout.value)

    # -- grids
    def _grid_len(self, which: int) -> int:
        i = self.get_info()
        if which == GRID_MARKER:
            return self.params.mpsi + 1
        return (i.P + 1) * i.mgrid * (3 if which == GRID_GRADPHI else 1)

    def get_grid(self, which: int) -> np.ndarray:
        n = self._grid_len(which)
        out = np.empty(n)
        self._chk(lib().gtcp_get_grid(self._h, which, n, _dp(out)), "get_grid")
        if which == GRID_MARKER:
            return out
        i = self.get_info()
        return out.reshape((i.P + 1, i.mgrid, 3) if which == GRID_GRADPHI else (i.P + 1, i.mgrid))

    def set_grid(self, which: int, arr: np.ndarray):
        a = np.ascontiguousarray(arr, dtype=np.float64).ravel()
        self._chk(lib().gtcp_set_grid(self._h, which, a.size, _dp(a)), "set_grid")

    # -- diagnostics
    def stats(self) -> dict:
        s = Stats()
        self._chk(lib().gtcp_stats(self._h, C.byref(s)), "stats")
        return {k: getattr(s, k) for k, _ in Stats._fields_}

    def diag(self) -> dict:
        d = Diag()
        self._chk(lib().gtcp_diag(self._h, C.byref(d)), "diag")
        return {k: getattr(d, k) for k, _ in Diag._fields_}

    def set_timing(self, on: bool = True):
        self._chk(lib().gtcp_set_timing(self._h, int(on)), "set_timing")

    def timings(self) -> dict:
        t = Timings()
        self._chk(lib().gtcp_timings(self._h, C.byref(t)), "timings")
        d = {f"{p}_ms": t.ms[i] for i, p in enumerate(PHASES)}
        d.update({f"{p}_calls": t.calls[i] for i, p in enumerate(PHASES)})
        d.update({f"{p}_comm_bytes": t.comm_bytes[i] for i, p in enumerate(PHASES)})
        d["launches"] = t.launches
        return d

    def timings_reset(self):
        self._chk(lib().gtcp_timings_reset(self._h), "timings_reset")

    def set_charge_mode(self, mode: int):
        self._chk(lib().gtcp_set_charge_mode(self._h, mode), "set_charge_mode")

    def set_push_mode(self, mode: int):
        self._chk(lib().gtcp_set_push_mode(self._h, mode), "set_push_mode")

    def set_fused(self, on: bool):
        self._chk(lib().gtcp_set_fused(self._h, int(bool(on))), "set_fused")


class LoopbackHub:
    """Test-only in-process transport (gtcp_loopback_create): nranks contexts
    of one process on one device share it instead of an NCCL id; drive each
    context from its own host thread on its own stream."""

    def __init__(self, nranks: int):
        self.handle = C.c_void_p()
        s = lib().gtcp_loopback_create(nranks, C.byref(self.handle))
        if s:
            raise GtcpError(s, "loopback_create")
        self.nranks = nranks

    def close(self):
        if self.handle and self.handle.value:
            lib().gtcp_loopback_destroy(self.handle)
            self.handle = C.c_void_p()


# module-level names matching the C ABI
def gtcp_init(params: Params, rank: int = 0, nranks: int = 1, nccl_id: bytes | None = None, stream=None) -> Context:
    return Context(params, rank, nranks, nccl_id, stream)


def gtcp_charge(ctx: Context): ctx.charge()
def gtcp_poisson_smooth(ctx: Context): ctx.poisson_smooth()
def gtcp_field(ctx: Context): ctx.field()
def gtcp_push(ctx: Context, stage: int): ctx.push(stage)
def gtcp_shift(ctx: Context): ctx.shift()
def gtcp_bin(ctx: Context): ctx.bin()
def gtcp_step(ctx: Context, nsteps: int = 1): ctx.step(nsteps)
def gtcp_load(ctx: Context): ctx.load()
def gtcp_set_particles(ctx: Context, parts: dict): ctx.set_particles(parts)
def gtcp_get_particles(ctx: Context) -> dict: return ctx.get_particles()
def gtcp_get_grid(ctx: Context, which: int): return ctx.get_grid(which)
def gtcp_set_grid(ctx: Context, which: int, arr): ctx.set_grid(which, arr)
def gtcp_stats(ctx: Context) -> dict: return ctx.stats()
def gtcp_destroy(ctx: Context): ctx.close()
