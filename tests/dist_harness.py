"""Decomposed-step parity harness (TEST INFRASTRUCTURE: uses the oracle).

Runs the GTC-P step decomposed over `world` ranks -- toroidal domains x
radial windows x particle replicas (§3.2) -- through the C ABI and
compares, step by step, with the oracle's single-domain step on the same
markers: particle count bit-exact, every particle inside its owner domain
(H-1 toroidal, H-2 radial: oracle.shift_dest / oracle.radial_dest), state and
stage-1 charge within the P-0 tolerance, one fixed-point scale on every rank.

Two transports drive the same harness:
  - LoopbackRanks: `world` contexts in ONE process on ONE GPU, one host thread
    and stream each, sharing a gtcp_loopback hub (pytest -m gpu on a 1-GPU box);
  - NcclRanks: one process per GPU under torchrun, NCCL inside libgtcp
    (tests/dist_parity.py).
"""
from __future__ import annotations

import math
from concurrent.futures import ThreadPoolExecutor

import numpy as np

import oracle
import paper_1510_05546_b200 as G
import synth

TWO_PI = 2 * math.pi
STATE = ("psi", "theta", "zeta", "rho", "w", "mu")


class LoopbackRanks:
    """`world` contexts of this process on the current GPU (gtcp_init_loopback)."""

    def __init__(self, params_of_rank):
        import torch
        self.world = len(params_of_rank)
        self.hub = G.LoopbackHub(self.world)
        self.streams = [torch.cuda.Stream() for _ in range(self.world)]
        self.pool = ThreadPoolExecutor(self.world)
        self.ctx = [None] * self.world

        def mk(r):
            torch.cuda.set_device(torch.cuda.current_device())
            self.ctx[r] = G.Context(params_of_rank[r], r, self.world, stream=self.streams[r].cuda_stream,
                                    loopback=self.hub)
        self.each(mk)

    def each(self, fn):
        """fn(rank) on every rank concurrently (their collectives meet in the hub)."""
        futs = [self.pool.submit(fn, r) for r in range(self.world)]
        return [f.result() for f in futs]

    def close(self):
        for c in self.ctx:
            if c is not None:
                c.close()
        self.hub.close()
        self.pool.shutdown()


class NcclRanks:
    """This process is one rank of a torchrun job; `each` gathers every rank's result."""

    def __init__(self, params_of_rank):
        import torch.distributed as dist
        self.dist = dist
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        obj = [G.gtcp_nccl_unique_id() if self.rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        self.ctx = {self.rank: G.Context(params_of_rank[self.rank], self.rank, self.world, obj[0])}

    def each(self, fn):
        out = [None] * self.world
        self.dist.all_gather_object(out, fn(self.rank))
        return out

    def close(self):
        self.ctx[self.rank].close()


def layout_params(size, world, npartdom=1, nradial=1, precision=64, **over):
    ntor = world // (npartdom * nradial)
    assert ntor * npartdom * nradial == world
    return [G.gtcp_default_params(size, ntoroidal=ntor, npartdom=npartdom, nradial=nradial, track_ids=1,
                                  bin_every=1, precision=precision, **over) for _ in range(world)]


def _round32(state):
    for k in STATE:
        state[k] = state[k].astype(np.float32).astype(np.float64)
    for k in ("theta", "zeta"):
        state[k] = np.where(state[k] >= TWO_PI, 0.0, state[k])


def run_parity(ranks, size, npartdom=1, nradial=1, precision=64, nparts=0, steps=2, w_amp=None, w_scale=None,
               seed=1, **over):
    """Returns a report dict with "ok".  w_scale(parts) may rescale weights per
    particle before the split (fixed-point scale agreement regressions)."""
    world = ranks.world
    ntor = world // (npartdom * nradial)
    cfg = synth.config(size, **over)
    p = oracle.make_params(cfg)
    g = oracle.geometry(p)
    P = cfg["mzetamax"] // ntor
    n = nparts or cfg["micell"] * (g.mgrid - cfg["mpsi"]) * cfg["mzetamax"]
    state = synth.load_particles(cfg, n, seed=seed, w_amp=w_amp)
    if w_scale is not None:
        w_scale(state)
    if precision == 32:  # the oracle sees the same fp32-rounded state
        _round32(state)
    tol = 1e-6 if precision == 64 else 1e-4

    def coords(r):
        return r // (npartdom * nradial), (r // npartdom) % nradial, r % npartdom

    def owner(st):
        t = oracle.shift_dest(p, st["zeta"], P)
        rr = oracle.radial_dest(p, st["psi"], nradial) if nradial > 1 else np.zeros(len(t), np.int32)
        return t, rr

    def distribute(st):
        t, rr = owner(st)
        sel = []
        for r in range(world):
            ct, cr, cp = coords(r)
            sel.append((t == ct) & (rr == cr) & ((st["id"] % npartdom) == cp))
        return sel

    sel = distribute(state)
    ranks.each(lambda r: ranks.ctx[r].set_particles({k: v[sel[r]] for k, v in state.items()}))
    nm = oracle.marker_norm(p, state)
    nm_gpu = ranks.each(lambda r: ranks.ctx[r].get_grid(G.GRID_MARKER))
    report = {"world": world, "ntoroidal": ntor, "nradial": nradial, "npartdom": npartdom, "size": size,
              "n": int(n), "precision": precision}
    report["marker_norm"] = max(float(np.max(np.abs(x - nm)) / np.max(np.abs(nm))) for x in nm_gpu)
    ok = report["marker_norm"] <= 1e-8
    for step in range(steps):
        def one_step(r):
            c = ranks.ctx[r]
            c.charge()
            rho = c.get_grid(G.GRID_CHARGE)
            fx1 = c.stats()["fx_shift"]
            c.poisson_smooth()
            c.field()
            c.push(1)
            c.shift()
            c.charge()
            fx2 = c.stats()["fx_shift"]
            c.poisson_smooth()
            c.field()
            c.push(2)
            c.shift()
            return rho, c.get_particles(STATE), c.stats(), (fx1, fx2)
        res = ranks.each(one_step)
        ch_ref = oracle.charge_global(p, state)
        oracle.step_global(p, state, nm)
        cat = {k: np.concatenate([x[1][k] for x in res]) for k in res[0][1]}
        o1, o2 = np.argsort(cat["id"]), np.argsort(state["id"])
        err = {"count": int(len(cat["id"]) == len(state["id"]) and np.array_equal(cat["id"][o1], state["id"][o2]))}
        if err["count"]:
            for k in ("psi", "rho", "w"):
                err[k] = float(np.max(np.abs(cat[k][o1] - state[k][o2])) / np.max(np.abs(state[k])))
            for k in ("theta", "zeta"):
                d = (cat[k][o1] - state[k][o2] + math.pi) % TWO_PI - math.pi
                err[k] = float(np.max(np.abs(d)) / TWO_PI)
        owner_ok = True
        for r, x in enumerate(res):
            t, rr = owner(x[1])
            ct, cr, _ = coords(r)
            owner_ok &= bool(np.all(t == ct)) and bool(np.all(rr == cr))
        err["owner"] = int(owner_ok)
        ce = 0.0
        for r, x in enumerate(res):  # every replica / radial window holds its toroidal domain's full charge
            t = coords(r)[0]
            ce = max(ce, float(np.max(np.abs(x[0][:P] - ch_ref[t * P:t * P + P]))))
        err["charge"] = ce / float(np.max(np.abs(ch_ref)))
        fxs = {x[3] for x in res}
        err["fx_shift_agree"] = int(len(fxs) == 1)
        err["movers_sent"] = int(sum(x[2]["movers_sent"] for x in res))
        report[f"step{step}"] = err
        keys = ("psi", "rho", "w", "theta", "zeta", "charge")
        ok &= err["count"] == 1 and err["owner"] == 1 and err["fx_shift_agree"] == 1 and \
            all(err.get(k, 1.0) <= tol for k in keys)
        # restart every rank from the oracle's state: identical inputs each step
        if precision == 32:
            _round32(state)
        sel = distribute(state)

        def reset(r):
            ranks.ctx[r].set_particles({k: v[sel[r]] for k, v in state.items()})
            ranks.ctx[r].set_grid(G.GRID_MARKER, nm)
        ranks.each(reset)
    report["ok"] = bool(ok)
    return report
