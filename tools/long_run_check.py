"""Long-run invariants under torchrun (N ranks): the global marker count is
conserved exactly and every marker stays inside its owner domain over many
steps of the decomposed step (shift + bin exercised repeatedly).

  torchrun --nproc-per-node 4 --master-addr 127.0.0.1 tools/long_run_check.py --size B --steps 100
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_1510_05546_b200 as G  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--size", default="B")
ap.add_argument("--steps", type=int, default=100)
ap.add_argument("--every", type=int, default=10)
ap.add_argument("--micell", type=int, default=20)
ap.add_argument("--nradial", type=int, default=1)
ap.add_argument("--npartdom", type=int, default=1)
a = ap.parse_args()
rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
nrad, npd = a.nradial, a.npartdom
ntor = world // (nrad * npd)
rank_t, rank_r = rank // (npd * nrad), (rank // npd) % nrad
p = G.gtcp_default_params(a.size, ntoroidal=ntor, nradial=nrad, npartdom=npd, micell=a.micell)
obj = [G.gtcp_nccl_unique_id() if rank == 0 else None]
dist.broadcast_object_list(obj, src=0)
ctx = G.Context(p, rank, world, obj[0])
ctx.load()
n0 = ctx.stats()["n_global"]
ok = True
rows = []
for s in range(a.every, a.steps + 1, a.every):
    ctx.step(a.every)
    st = ctx.stats()
    import numpy as np
    idx = np.random.default_rng(s).integers(0, max(st["n_local"], 1), size=min(4096, st["n_local"]))
    smp = ctx.sample_particles(idx, ("zeta", "psi"))
    P = p.mzetamax // ntor
    kg = np.minimum(np.floor(smp["zeta"] * (p.mzetamax / (2 * np.pi))), p.mzetamax - 1)
    inside = bool(np.all((kg // P) == rank_t)) and bool(np.all(np.isfinite(smp["zeta"])))
    if nrad > 1:  # G-6 equal-area windows snapped to rings (test-side restatement, as in dist_parity)
        dr = (p.a1 - p.a0) / p.mpsi
        rb = [min(max(int(np.floor((np.sqrt(p.a0**2 + k / nrad * (p.a1**2 - p.a0**2)) - p.a0) / dr + 0.5)), 0), p.mpsi)
              for k in range(1, nrad)]
        rbound = np.array([p.a0 + b * dr for b in rb])
        rd = np.sum(np.sqrt(2.0 * smp["psi"])[:, None] >= rbound[None, :], axis=1)
        inside = inside and bool(np.all(rd == rank_r))
    flag = torch.tensor([int(inside)], device="cuda")
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    good = st["n_global"] == n0 and int(flag.item()) == 1
    ok &= good
    if rank == 0:
        rows.append({"step": s, "n_global": st["n_global"], "n0": n0, "owners_ok": int(flag.item()), "ok": good,
                     "movers_sent": st.get("movers_sent")})
        print(json.dumps(rows[-1]), flush=True)
if rank == 0:
    print(json.dumps({"world": world, "ntoroidal": ntor, "nradial": nrad, "npartdom": npd, "size": a.size,
                      "steps": a.steps, "ok": bool(ok)}))
ctx.close()
dist.destroy_process_group()
sys.exit(0 if ok else 1)
