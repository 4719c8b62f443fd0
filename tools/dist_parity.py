"""Multi-GPU parity (torchrun, one rank per GPU, NCCL inside libgtcp):
the toroidally decomposed step against the oracle's single-domain step.

  torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/dist_parity.py --size T

Each rank loads the markers of its toroidal domain (host generator, global
ids), runs one full step through the C ABI, and rank 0 gathers all ranks'
particles and grids and compares them with the oracle (P-0 tolerances;
particle count bit-exact; every particle inside its owner domain)."""
import argparse
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--size", default="T")
ap.add_argument("--nparts", type=int, default=0, help="markers (0 = micell*(mgrid-mpsi)*mzetamax)")
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--w-amp", type=float, default=None)
ap.add_argument("--mzetamax", type=int, default=None)
ap.add_argument("--npartdom", type=int, default=1)
ap.add_argument("--nradial", type=int, default=1)
ap.add_argument("--precision", type=int, default=64)
a = ap.parse_args()

rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
import paper_1510_05546_b200 as G  # noqa: E402

over = {"mzetamax": a.mzetamax} if a.mzetamax else {}
cfg = synth.config(a.size, **over)
npd, nrad = a.npartdom, a.nradial
ntor = world // (npd * nrad)
rank_t, rank_r, rank_p = rank // (npd * nrad), (rank // npd) % nrad, rank % npd
params = G.gtcp_default_params(a.size, ntoroidal=ntor, npartdom=npd, nradial=nrad, track_ids=1, bin_every=1,
                                precision=a.precision, **over)
geo = G.gtcp_geometry(params)
n = a.nparts or cfg["micell"] * (geo["mgrid"] - cfg["mpsi"]) * cfg["mzetamax"]
parts = synth.load_particles(cfg, n, seed=1, w_amp=a.w_amp)
TOLP = 1e-6 if a.precision == 64 else 1e-4
if a.precision == 32:  # the oracle sees the same fp32-rounded state
    for _k in ("psi", "theta", "zeta", "rho", "w", "mu"):
        parts[_k] = parts[_k].astype(np.float32).astype(np.float64)
    for _k in ("theta", "zeta"):
        parts[_k] = np.where(parts[_k] >= 2 * math.pi, 0.0, parts[_k])
P = cfg["mzetamax"] // ntor
# G-6 radial windows: equal-area split snapped to the nearest ring (test-side restatement)
_dr = (cfg["a1"] - cfg["a0"]) / cfg["mpsi"]
_rb = [0]
for _k in range(1, nrad):
    _rk = math.sqrt(cfg["a0"] ** 2 + _k / nrad * (cfg["a1"] ** 2 - cfg["a0"] ** 2))
    _rb.append(min(max(int(math.floor((_rk - cfg["a0"]) / _dr + 0.5)), 0), cfg["mpsi"]))
_rb.append(cfg["mpsi"])
_rbound = np.array([cfg["a0"] + b * _dr for b in _rb])


def rdom(psi):
    r = np.sqrt(2.0 * psi)
    return np.sum(r[:, None] >= _rbound[None, 1:nrad], axis=1) if nrad > 1 else np.zeros(len(psi), np.int64)

cz = cfg["mzetamax"] / (2.0 * math.pi)
kg = np.minimum(np.floor(parts["zeta"] * cz).astype(np.int64), cfg["mzetamax"] - 1)
mine = ((kg // P) == rank_t) & (rdom(parts["psi"]) == rank_r) & ((parts["id"] % npd) == rank_p)
obj = [G.gtcp_nccl_unique_id() if rank == 0 else None]
dist.broadcast_object_list(obj, src=0)
ctx = G.Context(params, rank, world, obj[0])
ctx.set_particles({k: v[mine] for k, v in parts.items()})


def gather_all(d):
    out = [None] * world
    dist.all_gather_object(out, d)
    return out


report = {}
ok = True
orc_state = {k: v.copy() for k, v in parts.items()}
import oracle  # noqa: E402  (test infrastructure: this script is a parity harness)
p = oracle.make_params(cfg)
nm = oracle.marker_norm(p, orc_state) if rank == 0 else None
obj = [nm]
dist.broadcast_object_list(obj, src=0)
nm = obj[0]
nm_gpu = ctx.get_grid(G.GRID_MARKER)  # computed by the library (ring sums allreduced over ranks)
report["marker_norm"] = float(np.max(np.abs(nm_gpu - nm)) / np.max(np.abs(nm)))
ok &= report["marker_norm"] <= 1e-8
for step in range(a.steps):
    ctx.charge()
    rho = ctx.get_grid(G.GRID_CHARGE)
    ctx.poisson_smooth()
    ctx.field()
    ctx.push(1)
    ctx.shift()
    ctx.charge()
    ctx.poisson_smooth()
    ctx.field()
    ctx.push(2)
    ctx.shift()
    got = ctx.get_particles(("psi", "theta", "zeta", "rho", "w", "mu"))
    allp = gather_all(got)
    allrho = gather_all(rho)
    st = ctx.stats()
    if rank == 0:
        # oracle: one step on the single global domain, from the same state
        ch_ref = oracle.charge_global(p, orc_state)
        oracle.step_global(p, orc_state, nm)
        cat = {k: np.concatenate([x[k] for x in allp]) for k in allp[0]}
        o1, o2 = np.argsort(cat["id"]), np.argsort(orc_state["id"])
        err = {}
        err["count"] = int(len(cat["id"]) == len(orc_state["id"]) and np.array_equal(cat["id"][o1], orc_state["id"][o2]))
        for k in ("psi", "rho", "w"):
            err[k] = float(np.max(np.abs(cat[k][o1] - orc_state[k][o2])) / np.max(np.abs(orc_state[k])))
        for k in ("theta", "zeta"):
            d = (cat[k][o1] - orc_state[k][o2] + math.pi) % (2 * math.pi) - math.pi
            err[k] = float(np.max(np.abs(d)) / (2 * math.pi))
        # every particle inside its owner domain
        owner_ok = True
        for r, x in enumerate(allp):
            kk = np.minimum(np.floor(x["zeta"] * cz).astype(np.int64), cfg["mzetamax"] - 1)
            owner_ok &= bool(np.all(kk // P == r // (npd * nrad)))
            owner_ok &= bool(np.all(rdom(x["psi"]) == (r // npd) % nrad))
        err["owner"] = int(owner_ok)
        # stage-1 charge on planes [r*P, r*P+P] of each rank vs the oracle's global grid
        ce = 0.0
        for r, g in enumerate(allrho):
            t = r // (npd * nrad)  # every replica / radial domain holds the full charge of its toroidal domain
            ce = max(ce, float(np.max(np.abs(g[:P] - ch_ref[t * P:t * P + P]))))
        err["charge"] = ce / float(np.max(np.abs(ch_ref)))
        err["movers_sent"] = int(st["movers_sent"])
        report[f"step{step}"] = err
        ok &= err["count"] == 1 and err["owner"] == 1 and all(err[k] <= TOLP for k in ("psi", "rho", "w", "theta", "zeta", "charge"))
        # continue both sides from the oracle state (identical inputs each step)
    # reset every rank to the oracle trajectory for the next step
    obj = [orc_state if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    st_all = obj[0]
    if rank != 0:
        orc_state = st_all
    if a.precision == 32:  # the library stores fp32: restart both sides from the rounded state
        for _k in ("psi", "theta", "zeta", "rho", "w", "mu"):
            st_all[_k] = st_all[_k].astype(np.float32).astype(np.float64)
        for _k in ("theta", "zeta"):
            st_all[_k] = np.where(st_all[_k] >= 2 * math.pi, 0.0, st_all[_k])
        orc_state = st_all
    zz = np.minimum(np.floor(st_all["zeta"] * cz).astype(np.int64), cfg["mzetamax"] - 1)
    sel = ((zz // P) == rank_t) & (rdom(st_all["psi"]) == rank_r) & ((st_all["id"] % npd) == rank_p)
    ctx.set_particles({k: v[sel] for k, v in st_all.items()})
    ctx.set_grid(G.GRID_MARKER, nm)
if rank == 0:
    print(json.dumps({"world": world, "ntoroidal": ntor, "nradial": nrad, "npartdom": npd, "size": a.size, "n": int(n), "ok": bool(ok), **report}))
ctx.close()
dist.destroy_process_group()
sys.exit(0 if (rank != 0 or ok) else 1)
