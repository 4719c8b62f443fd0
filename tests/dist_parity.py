"""Multi-GPU parity (torchrun, one rank per GPU, NCCL inside libgtcp): the
decomposed step against the oracle's single-domain step (tests/dist_harness.py).

  torchrun --nproc-per-node N --master-addr 127.0.0.1 tests/dist_parity.py --size T --mzetamax 8

Rank 0 prints one JSON report; exit status 0 iff it is ok.  The same harness
runs on one GPU through the loopback transport (tests/test_gpu_loopback.py)."""
import argparse
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import dist_harness as H  # noqa: E402

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
over = {"mzetamax": a.mzetamax} if a.mzetamax else {}
ranks = H.NcclRanks(H.layout_params(a.size, world, a.npartdom, a.nradial, a.precision, **over))
rep = H.run_parity(ranks, a.size, a.npartdom, a.nradial, a.precision, a.nparts, a.steps, a.w_amp, **over)
if rank == 0:
    print(json.dumps(rep), flush=True)
ranks.close()
dist.destroy_process_group()
sys.exit(0 if (rank != 0 or rep["ok"]) else 1)
