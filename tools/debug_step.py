"""Debug driver: a few steps at a small size on one GPU (run with
GTCP_LIB_PATH pointing at a -DGTCP_DEBUG build to get device asserts)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1510_05546_b200 as G
import synth
size = sys.argv[1] if len(sys.argv) > 1 else "T"
mz = int(sys.argv[2]) if len(sys.argv) > 2 else 8
n = int(sys.argv[3]) if len(sys.argv) > 3 else 50000
cfg = synth.config(size, mzetamax=mz)
parts = synth.load_particles(cfg, n, seed=1)
ctx = G.Context(G.gtcp_default_params(size, mzetamax=mz, track_ids=1))
ctx.set_particles(parts)
print("set ok", flush=True)
ctx.charge(); ctx.get_grid(G.GRID_CHARGE); print("charge ok", flush=True)
ctx.poisson_smooth(); ctx.field(); ctx.get_grid(G.GRID_PHI); print("field ok", flush=True)
ctx.push(1); ctx.stats(); print("push1 ok", flush=True)
ctx.shift(); ctx.charge(); ctx.stats(); print("charge2 ok", flush=True)
ctx.poisson_smooth(); ctx.field(); ctx.push(2); ctx.shift(); ctx.stats(); print("step ok", flush=True)
ctx.step(3); print("3 steps ok", ctx.stats()["n_global"], flush=True)
