"""Small driver for compute-sanitizer (memcheck / racecheck / synccheck):
config T, two full steps with a bin, the tiled and the direct deposit, the
grid kernels, push, diagnostics; then config T with 8 planes and the shift
path exercised through two loopback ranks.

  compute-sanitizer --tool memcheck python tools/sanitize_run.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402

import paper_1510_05546_b200 as G  # noqa: E402
import synth  # noqa: E402

cfg = synth.config("T")
parts = synth.load_particles(cfg, 12100, seed=1, w_amp=0.05)
ctx = G.Context(G.gtcp_default_params("T", track_ids=1, bin_every=1))
ctx.set_particles(parts)
ctx.step(2)
ctx.set_charge_mode(1)
ctx.step(1)
ctx.charge()
ctx.poisson_smooth()
ctx.field()
d = ctx.diag()
st = ctx.stats()
ctx.close()
print("single-rank ok", st["n_global"], d["field_energy"] > 0, flush=True)

import dist_harness as H  # noqa: E402  (loopback ranks: shift, ghost planes, allreduces)
ranks = H.LoopbackRanks(H.layout_params("T", 2, mzetamax=8))
cfg8 = synth.config("T", mzetamax=8)
p8 = synth.load_particles(cfg8, 12000, seed=3)
kg = np.minimum(np.floor(p8["zeta"] * 8 / (2 * np.pi)).astype(int), 7)


def go(r):
    c = ranks.ctx[r]
    c.set_particles({k: v[(kg // 4) == r] for k, v in p8.items()})
    c.step(2)
    return c.stats()["n_global"]


print("loopback ok", ranks.each(go), flush=True)
ranks.close()
