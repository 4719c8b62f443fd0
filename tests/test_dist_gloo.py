"""World-size-2 `gloo` tests (CPU) of the multi-rank host logic of the toroidal
decomposition: domain ownership (H-1), the shift protocol that
libgtcp implements with NCCL (count exchange, left/right payloads straight
behind the keepers, multi-hop passes with a guard, H-3), and bench.py's
max-over-ranks timing.  The GPU path itself is covered by
tests/test_gpu_parity.py::test_toroidal_decomposition_parity_2gpu."""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth

TWO_PI = 2 * math.pi


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _dest(zeta, mzetamax, P):
    # H-1: same expression as the oracle / the CUDA classify (one rounded multiply)
    import oracle
    cfg = synth.config("T", mzetamax=mzetamax)
    return oracle.shift_dest(oracle.make_params(cfg), zeta, P)


def _shift(parts, rank, world, mzetamax):
    """Reference of libgtcp's shift_exchange: classify (shorter way round),
    send left/right, receive right-then-left, append behind the keepers,
    re-check arrivals only, guard = world passes."""
    P = mzetamax // world
    left, right = (rank - 1) % world, (rank + 1) % world
    start = 0
    for _ in range(world + 1):
        tail = {k: v[start:] for k, v in parts.items()}
        d = _dest(tail["zeta"], mzetamax, P)
        rel = (d - rank) % world
        cls = np.where(rel == 0, 0, np.where(rel <= world // 2, 2, 1))
        counts = torch.tensor([int((cls == 1).sum()), int((cls == 2).sum())], dtype=torch.int64)
        tot = counts.sum().clone()
        dist.all_reduce(tot)
        if int(tot) == 0:
            break
        recv_from_right = torch.zeros(1, dtype=torch.int64)
        recv_from_left = torch.zeros(1, dtype=torch.int64)
        reqs = [dist.isend(counts[0:1].clone(), left), dist.isend(counts[1:2].clone(), right),
                dist.irecv(recv_from_right, right), dist.irecv(recv_from_left, left)]
        for r in reqs:
            r.wait()
        keep = {k: v[cls == 0] for k, v in tail.items()}
        outL = {k: v[cls == 1] for k, v in tail.items()}
        outR = {k: v[cls == 2] for k, v in tail.items()}
        newtail = {}
        for k in tail:
            a = torch.from_numpy(np.ascontiguousarray(outL[k]).astype(np.float64))
            b = torch.from_numpy(np.ascontiguousarray(outR[k]).astype(np.float64))
            fr = torch.zeros(int(recv_from_right), dtype=torch.float64)
            fl = torch.zeros(int(recv_from_left), dtype=torch.float64)
            reqs = [dist.isend(a, left), dist.isend(b, right), dist.irecv(fr, right), dist.irecv(fl, left)]
            for r in reqs:
                r.wait()
            newtail[k] = np.concatenate([keep[k], fr.numpy(), fl.numpy()]).astype(parts[k].dtype)
        nkeep = len(keep["zeta"])
        parts = {k: np.concatenate([parts[k][:start], newtail[k]]) for k in parts}
        start = start + nkeep
    return parts


def _worker(rank, world, port, mzetamax, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = synth.config("T", mzetamax=mzetamax)
        P = mzetamax // world
        allp = synth.load_particles(cfg, 4000, seed=3)
        allp["id"] = allp["id"].astype(np.float64)
        # owned set by H-1
        d = _dest(allp["zeta"], mzetamax, P)
        mine = {k: v[d == rank] for k, v in allp.items()}
        # move every particle by a random toroidal displacement (up to 1.6 domains, multi-hop)
        rng = np.random.default_rng(rank)
        z = mine["zeta"] + rng.uniform(-1.6, 1.6, len(mine["zeta"])) * TWO_PI / world
        mine["zeta"] = z - TWO_PI * np.floor(z / TWO_PI)
        n0 = torch.tensor([len(mine["zeta"])], dtype=torch.float64)
        w0 = torch.tensor([mine["w"].sum()], dtype=torch.float64)
        dist.all_reduce(n0)
        dist.all_reduce(w0)
        out = _shift(mine, rank, world, mzetamax)
        n1 = torch.tensor([len(out["zeta"])], dtype=torch.float64)
        w1 = torch.tensor([out["w"].sum()], dtype=torch.float64)
        dist.all_reduce(n1)
        dist.all_reduce(w1)
        owner_ok = bool(np.all(_dest(out["zeta"], mzetamax, P) == rank))
        second = _shift(out, rank, world, mzetamax)
        # max-over-ranks timing as bench.py does it
        t = torch.tensor([10.0 + rank], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        q.put((rank, float(n0), float(n1), float(w0), float(w1), owner_ok,
               len(second["zeta"]) == len(out["zeta"]), float(t)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mzetamax", [4, 8])
def test_shift_protocol_world2(orc, mzetamax):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mzetamax, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, n0, n1, w0, w1, owner_ok, idem, t in res:
        assert n0 == n1                        # particle count bit-exact (H-3)
        assert abs(w0 - w1) <= 1e-12 * max(1.0, abs(w0))
        assert owner_ok                        # everybody inside its owner domain
        assert idem                            # a second shift moves nobody
        assert t == 11.0                       # max over ranks
