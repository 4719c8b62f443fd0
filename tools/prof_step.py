"""Short profiling / timing driver: load a class, run warm-up + timed steps,
print per-phase CUDA-event times (ms per step).  Used for ncu captures and
A/B experiments (env knobs: GTCP_DEPOSIT_CTAS, GTCP_PROFILE_BIN, GTCP_PROFILE_SHIFT)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

ap = argparse.ArgumentParser()
ap.add_argument("--size", default="A")
ap.add_argument("--steps", type=int, default=1)
ap.add_argument("--warmup", type=int, default=0)
ap.add_argument("--charge-mode", type=int, default=0)
ap.add_argument("--bin-every", type=int, default=3)
ap.add_argument("--tag", default="")
ap.add_argument("--micell", type=int, default=None)
ap.add_argument("--bin-mu", type=int, default=None)
ap.add_argument("--mzetamax", type=int, default=None)
ap.add_argument("--precision", type=int, default=64)
ap.add_argument("--field-f32", type=int, default=0)
ap.add_argument("--fused", type=int, default=0)
a = ap.parse_args()

import torch  # noqa: E402

import paper_1510_05546_b200 as G  # noqa: E402

torch.cuda.set_device(0)
over = {"micell": a.micell} if a.micell else {}
if a.bin_mu:
    over["bin_mu"] = a.bin_mu
if a.mzetamax:
    over["mzetamax"] = a.mzetamax
over["precision"] = a.precision
over["field_f32"] = a.field_f32
stream = torch.cuda.Stream()
ctx = G.Context(G.gtcp_default_params(a.size, bin_every=a.bin_every, **over), stream=stream.cuda_stream)
ctx.set_charge_mode(a.charge_mode)
if a.fused:
    ctx.set_fused(True)
ctx.load()
ctx.step(a.warmup)
ctx.set_timing(True)
ctx.timings_reset()
ctx.step(a.steps)
t = ctx.timings()
st = ctx.stats()
out = {"tag": a.tag, "size": a.size, "steps": a.steps}
out.update({k: round(v / max(a.steps, 1), 3) for k, v in t.items() if k.endswith("_ms")})
out.update({k: st[k] for k in ("n_local", "charge_global_fallback", "fx_shift", "reflections")})
print(json.dumps(out))
