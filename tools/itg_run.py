"""ITG demonstration: a nonlinear delta-f run on a class-A
grid, printing the field energy sum(phi^2) and max|w| every `--every` steps.
Linear ITG growth shows as a straight line in log(energy) until saturation.

  python tools/itg_run.py --steps 400 --every 20 --micell 20
"""
import argparse
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1510_05546_b200 as G  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--size", default="A")
ap.add_argument("--steps", type=int, default=400)
ap.add_argument("--every", type=int, default=20)
ap.add_argument("--micell", type=int, default=20)
ap.add_argument("--w-amp", type=float, default=1e-3)
a = ap.parse_args()
torch.cuda.set_device(0)
p = G.gtcp_default_params(a.size, micell=a.micell, w_init_amp=a.w_amp)
ctx = G.Context(p)
ctx.load()
rows = []
for s in range(0, a.steps + 1, a.every):
    if s:
        ctx.step(a.every)
    ctx.charge()  # diagnostics only: the field of the current state
    ctx.poisson_smooth()
    phi = ctx.get_grid(G.GRID_PHI)
    st = ctx.stats()
    e = float(np.sum(phi * phi))
    rows.append({"step": s, "t": s * p.dt, "field_energy": e, "log_e": math.log(e) if e > 0 else None,
                 "max_abs_w": st["max_abs_w"], "n": st["n_global"]})
    print(json.dumps(rows[-1]), flush=True)
