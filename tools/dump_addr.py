"""Debug: dump the lo-limb ATOMS word offsets of sampled tiles of one
k_deposit_tiled launch and count the wavefronts per instruction (max distinct
words on one bank).  Needs the debug build:
  python paper_1510_05546_b200/_build.py -DGTCP_DUMP_ADDR --out=$PWD/paper_1510_05546_b200/_lib/libgtcp_dump.so
  GTCP_LIB_PATH=$PWD/paper_1510_05546_b200/_lib/libgtcp_dump.so python tools/dump_addr.py A
Note: ATOMS.ADD lanes on the same word serialise (each carries its own value);
the microbenchmark's constant increments compile to ATOMS.POPC.INC, which
merges them, so replaying these offsets (tools/microbench/replay.cu) gives
the distinct-word count, a lower bound."""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1510_05546_b200 as G  # noqa: E402

size = sys.argv[1] if len(sys.argv) > 1 else "A"
over = {"mzetamax": int(sys.argv[2])} if len(sys.argv) > 2 else {}
torch.cuda.set_device(0)
ctx = G.Context(G.gtcp_default_params(size, **over))
ctx.load()
ctx.step(1)
ctx.charge()
torch.cuda.synchronize()
buf = np.zeros(64 * 8 * 8 * 32 * 32, np.uint32)
G.lib().gtcp_debug_addr_dump(buf.ctypes.data_as(ctypes.POINTER(ctypes.c_uint)))
a = buf.reshape(64, 8, 8, 32, 32)
wf, dist = [], []
for t in range(64):
    for it in range(8):
        for w in range(8):
            for ins in range(32):
                x = a[t, it, w, ins]
                if not x.any():
                    continue
                u = np.unique(x)
                wf.append(np.bincount(u % 32, minlength=32).max())
                dist.append(len(u))
sel = [x for x in a.reshape(-1, 32) if x.any()]
np.array(sel, np.uint32).tofile(f"gpurun_out/addr_{size}.bin")
print(size, over, "instr", len(wf), "wavefronts/ATOMS %.2f" % np.mean(wf), "distinct words/instr %.1f" % np.mean(dist))
