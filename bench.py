"""Benchmark: particle-steps/s of the GTC-P hot path (BASELINE.json metric).

  python bench.py --gpus N --steps K --warmup W [--impl reference] [--size A]

One step = gtcp_step(1): two RK2 stages of charge, poisson_smooth, field,
push, shift (+ bin on schedule).  N = 1 runs GTC-P class A (configs[1]:
mpsi=90, mthetamax=640, mzetamax=64, micell=100, 207,097,600 markers) on one
B200.  N > 1 (torchrun, one rank per GPU, NCCL) runs class B toroidally
decomposed over N GPUs (configs[2]).  `value` is the whole-job throughput over
the full timed step (LIGHT grid kernels included); the charge+push+shift
phase times are reported beside it.  `--impl reference` times the CPU oracle
(oracle/, single thread) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "particle-steps/sec (charge+push+shift) at 1/2/4/8 B200; % HBM roofline"
UNIT = "particle-steps/s"
S = 8  # bytes per real (fp64)
# algorithmic bytes per particle: charge 5S/stage; push stage 1
# 11S (6S read + 5S write), stage 2 16S (11S read + 5S write)
BYTES = {"charge": 5 * S, "push1": 11 * S, "push2": 16 * S}


def peaks():
    try:
        d = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, smax, reasons = [], 0.0, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for l in self.lines:
            f = [x.strip() for x in l.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = max(smax, float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def host_info() -> dict:
    """nproc and the CPU model of the box the oracle runs on."""
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return {"nproc": os.cpu_count(), "lscpu_model": model}


def cpu_baseline(size: str, n_sample: int, steps: int = 1, parallel: bool = True):
    """Oracle (C, fp64) charge + push + shift on a bounded sample of the
    workload's markers, on the workload's full grid, with a fixed prescribed
    field.  parallel: the paper's CPU method on all host cores (OpenMP threads
    over particle ranges, per-thread grid replicas summed in a fixed order,
    P:330); else one thread.  Returns (particle-steps/s, seconds, threads)."""
    import numpy as np

    import oracle
    import synth
    cfg = synth.config(size)
    p = oracle.make_params(cfg)
    g = oracle.geometry(p)
    parts = synth.load_particles(cfg, n_sample, seed=2)
    K = cfg["mzetamax"]
    rng = np.random.default_rng(0)
    gp = 1e-3 * rng.standard_normal((K + 1, g.mgrid, 3))
    Xa = {k: parts[k].copy() for k in oracle.ATTRS}
    Xb = {k: v.copy() for k, v in Xa.items()}
    dep = oracle.deposit_replicas if parallel else oracle.deposit
    push = oracle.push_omp if parallel else oracle.push
    dest = oracle.shift_dest_omp if parallel else oracle.shift_dest
    t0 = time.perf_counter()
    for _ in range(steps):
        for stage in (1, 2):
            cur = dict(Xa if stage == 1 else Xb, mu=parts["mu"])
            grid, _ = dep(p, cur)
            oracle.charge_reduce_global(p, grid)
            push(p, stage, Xa, Xb, parts["mu"], gp)
            dest(p, (Xb if stage == 1 else Xa)["zeta"], K)
    dt = time.perf_counter() - t0
    return n_sample * steps / dt, dt, (oracle.omp_threads() if parallel else 1)


def workload_config(size: str, n_gpus: int, args) -> dict:
    """The workload both arms report (same keys and strings): class, grid,
    marker count, decomposition."""
    import synth
    over = {"micell": args.micell} if args.micell else {}
    if args.mzetamax:
        over["mzetamax"] = args.mzetamax
    cfg = synth.config(size, **over)
    # grid size from the product's host geometry (G-1..G-2); no oracle here
    import paper_1510_05546_b200 as G
    mgrid = G.gtcp_geometry(G.gtcp_default_params(size, **over))["mgrid"]
    ntor = max(1, n_gpus // (args.nradial * args.npartdom))
    return {"workload": f"GTC-P class {size}: mpsi={cfg['mpsi']} mthetamax={cfg['mthetamax']} "
                        f"mzetamax={cfg['mzetamax']} micell={cfg['micell']}",
            "particles": int(cfg["micell"] * (mgrid - cfg["mpsi"]) * cfg["mzetamax"]),
            "grid_nodes_per_plane": int(mgrid), "planes": cfg["mzetamax"],
            "decomposition": f"{ntor} toroidal x {args.nradial} radial x {args.npartdom} particle"}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    size = args.size or ("A" if args.gpus == 1 else "B")  # the same workload as the b200 arm
    n_sample = args.ref_sample
    import oracle
    oracle.build()
    vals = []
    for i in range(args.warmup + args.steps):
        v, dt, nthr = cpu_baseline(size, n_sample, 1)
        if i >= args.warmup:
            vals.append((v, dt))
    total_t = sum(dt for _, dt in vals)
    value = n_sample * len(vals) / total_t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total_t / len(vals),
        "higher_is_better": True, "scaling": "strong" if args.gpus > 1 else "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": workload_config(size, args.gpus, args),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": nthr, "kind": "oracle",
                         "sample": f"{n_sample} markers of class {size} on its full grid, charge+push+shift, "
                                   f"fixed prescribed field, {len(vals)} steps; OpenMP over {nthr} threads with "
                                   f"per-thread grid replicas summed in a fixed order (P:330)",
                         "host": host_info()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_gpu(args):
    import numpy as np
    import torch

    import paper_1510_05546_b200 as G

    rank, world, local = dist_env()
    assert world == args.gpus, f"--gpus {args.gpus} but WORLD_SIZE={world}"
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    size = args.size or ("A" if world == 1 else "B")
    over = {"micell": args.micell} if args.micell else {}
    if args.mzetamax:
        over["mzetamax"] = args.mzetamax
    ntor = world // (args.nradial * args.npartdom)
    assert ntor * args.nradial * args.npartdom == world, "GPUs must equal ntoroidal * nradial * npartdom"
    p = G.gtcp_default_params(size, ntoroidal=ntor, nradial=args.nradial, npartdom=args.npartdom,
                              bin_every=args.bin_every, precision=args.precision, **over)
    if args.bin_mu:
        p.bin_mu = args.bin_mu
    nccl_id = None
    if world > 1:
        obj = [G.gtcp_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    stream = torch.cuda.Stream()
    ctx = G.Context(p, rank, world, nccl_id, stream.cuda_stream)
    if args.push_mode:
        ctx.set_push_mode(args.push_mode)  # ablation: loop fission
    if args.charge_mode:
        ctx.set_charge_mode(args.charge_mode)  # ablation: global-atomic deposit
    if args.fused:
        ctx.set_fused(True)  # push + next-stage deposit in one kernel
    ctx.load()
    info = ctx.get_info()
    n_local = info.n_local
    n_total = n_local
    if world > 1:
        t = torch.tensor([n_local], dtype=torch.int64, device="cuda")
        dist.all_reduce(t)
        n_total = int(t.item())

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
            torch.cuda.synchronize()

    # warm-up
    for _ in range(args.warmup):
        ctx.step(1)
    ctx.set_timing(True)
    ctx.timings_reset()
    launches0 = ctx.timings()["launches"]
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    barrier()
    sync_t = torch.zeros(1, device="cuda")
    with ClockSampler(local) as clk:
        if dist:
            # device-side start line: a collective on the context stream right
            # before the start event, so host launch skew after the barrier is
            # not counted as step time on the ranks that wait for the others
            with torch.cuda.stream(stream):
                dist.all_reduce(sync_t)
        ev0.record(stream)
        for _ in range(args.steps):
            ctx.step(1)
        ev1.record(stream)
        torch.cuda.synchronize()
    barrier()
    ms = ev0.elapsed_time(ev1)
    tm = ctx.timings()
    launches = tm["launches"] - launches0
    if os.environ.get("BENCH_RANK_PHASES"):  # diagnostics: per-rank phase sum vs own elapsed
        ph = {k[:-3]: round(tm[k] / args.steps, 2) for k in tm if k.endswith("_ms")}
        print(f"[rank {rank}] own {ms / args.steps:.2f} ms/step, phases {sum(ph.values()):.2f}: {ph}",
              file=sys.stderr, flush=True)
    if dist:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = n_total * args.steps / (ms * 1e-3)
    cps_ms = tm["charge_ms"] + tm["charge_red_ms"] + tm["push_ms"] + tm["shift_ms"] + tm["bin_ms"]
    hbm, peak_kind = peaks()
    # roofline of the per-stage kernels: algorithmic bytes / average launch time
    roof = {}
    for name, ms_tot, calls, nbytes in (
            ("charge_deposit", tm["charge_ms"], tm["charge_calls"], BYTES["charge"]),
            ("push", tm["push_ms"], tm["push_calls"], 0.5 * (BYTES["push1"] + BYTES["push2"]))):
        if calls:
            avg_ms = ms_tot / calls
            gbs = n_local * nbytes / (avg_ms * 1e-3) / 1e9
            roof[name] = {"avg_ms": avg_ms, "achieved_gbs": gbs, "frac": gbs / hbm,
                          "bytes_per_particle": nbytes, "share_of_step": ms_tot / max(ms, 1e-9)}
    dom = max(roof, key=lambda k: roof[k]["share_of_step"]) if roof else None
    # inter-GPU bytes the library moved per phase (NCCL bus-byte convention,
    # counted in libgtcp), over that phase's event time: a lower bound of the
    # link rate, since each phase also holds the kernels around its collectives
    comm = {}
    for ph in ("charge", "charge_red", "poisson", "shift"):
        b = tm.get(f"{ph}_comm_bytes", 0)
        if b:
            t_ms = tm[f"{ph}_ms"]
            comm[ph] = {"bytes_per_step": b / args.steps, "ms_per_step": t_ms / args.steps,
                        "gbs_over_phase": b / (t_ms * 1e-3) / 1e9 if t_ms else None}
    if comm:
        comm["nvlink_ref_gbs"] = {"peer_copy_per_direction": 770, "nominal_per_direction": 900,
                                  "source": "/opt/skills/guides/B200_PROFILING.md (measured on this pool)"}
    traffic = None
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        traffic = tr.get(size, {}).get(dom)
        # the deposit's own roof: shared-memory atomic wavefronts (one per clock
        # per SM; ncu count per launch at this configuration) over its live time
        wf = tr.get(size, {}).get("charge_deposit", {}).get("smem_atomic_wavefronts_per_launch")
        if wf and "charge_deposit" in roof:
            props = torch.cuda.get_device_properties(local)
            clk_hz = (clk.summary() or {}).get("sm_mhz") or 1965.0
            peak_wf = props.multi_processor_count * clk_hz * 1e6
            ach = wf / (roof["charge_deposit"]["avg_ms"] * 1e-3)
            roof["charge_deposit"]["smem_atomic"] = {
                "achieved_wavefronts_per_s": ach, "peak_wavefronts_per_s": peak_wf, "frac": ach / peak_wf,
                "wavefronts_per_launch": wf, "source": "ncu l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom"}
        # both kernels' own roof: the L1/shared data pipe (one wavefront per clock
        # per SM), all its wavefronts (global gathers, shared atomics and loads)
        for kern in ("charge_deposit", "push"):
            wfa = tr.get(size, {}).get(kern, {}).get("l1_data_pipe_wavefronts_per_launch")
            if wfa and kern in roof:
                props = torch.cuda.get_device_properties(local)
                clk_hz = (clk.summary() or {}).get("sm_mhz") or 1965.0
                peak_wf = props.multi_processor_count * clk_hz * 1e6
                ach = wfa / (roof[kern]["avg_ms"] * 1e-3)
                roof[kern]["l1_data_pipe"] = {
                    "achieved_wavefronts_per_s": ach, "peak_wavefronts_per_s": peak_wf, "frac": ach / peak_wf,
                    "wavefronts_per_launch": wfa, "source": "ncu l1tex__data_pipe_lsu_wavefronts (lgds + shared)"}
    except Exception:
        pass
    # end to end through the C ABI with HOST buffers (pinned): H2D state, step, D2H state
    e2e = None
    if not args.no_e2e:
        k_e2e = max(1, min(args.steps, args.e2e_steps))
        parts = ctx.get_particles(("psi", "theta", "zeta", "rho", "w", "mu"))
        n_e2e = len(parts["psi"])
        cap = ctx.get_info().capacity  # the owned count may change under a decomposed run
        host = []
        for k in ("psi", "theta", "zeta", "rho", "w", "mu"):
            a = torch.empty(cap, dtype=torch.float64).pin_memory().numpy()
            a[:n_e2e] = parts[k]
            host.append(a)
        del parts
        ctx.set_timing(False)
        barrier()
        t0 = time.perf_counter()
        h2d = d2h = 0
        for _ in range(k_e2e):
            h2d += 6 * 8 * n_e2e
            n_e2e = ctx.step_host(host, 1, n_e2e)
            d2h += 6 * 8 * n_e2e
        barrier()
        dt = time.perf_counter() - t0
        if dist:
            t = torch.tensor([dt], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        if dist:
            t = torch.tensor([h2d, d2h], dtype=torch.int64, device="cuda")
            dist.all_reduce(t)
            h2d, d2h = int(t[0].item()), int(t[1].item())
        e2e = {"value": n_total * k_e2e / dt, "unit": UNIT, "h2d_bytes_per_step": h2d // k_e2e,
               "d2h_bytes_per_step": d2h // k_e2e, "steps": k_e2e,
               "how": "gtcp_step_host: pinned host SoA (live state + mu) -> device, one step, "
                      "device -> host (live state + mu), per step, all ranks"}
    out = None
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu:
            v, dt, nthr = cpu_baseline(size, args.ref_sample, 1, parallel=True)
            v1, dt1, _ = cpu_baseline(size, args.ref_sample // 8, 1, parallel=False)
            cpu = {"value": v, "unit": UNIT, "cores": nthr, "kind": "oracle",
                   "sample": f"{args.ref_sample} markers of class {size} on its full grid, one step of "
                             f"charge+push+shift with a fixed field ({dt:.1f} s on {nthr} OpenMP threads, "
                             f"per-thread grid replicas summed in a fixed order, P:330)",
                   "single_thread": {"value": v1, "sample": f"{args.ref_sample // 8} markers, {dt1:.1f} s"},
                   "host": host_info()}
        r = roof.get(dom, {})
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "f64",
            "state_storage": "f64" if args.precision == 64 else "f32 (arithmetic f64)",
            "data": "synthetic",
            "config": dict(workload_config(size, world, args), micell=p.micell, bin_every=p.bin_every,
                           l2="inputs larger than L2 (particle SoA %.1f GB/GPU)"
                              % (n_local * 11 * (8 if args.precision == 64 else 4) / 1e9)),
            "value_charge_push_shift": n_total * args.steps / (cps_ms * 1e-3) if cps_ms else None,
            "phase_ms_per_step": {k[:-3]: tm[k] / args.steps for k in tm if k.endswith("_ms")},
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": r.get("achieved_gbs"), "peak": hbm,
                         "peak_kind": peak_kind, "unit": "GB/s", "frac": r.get("frac"), "traffic": traffic,
                         "all": roof},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clk.summary(),
        }
        if world > 1:
            out["comm"] = comm
        variant = [f"charge_mode {args.charge_mode}"] * bool(args.charge_mode) + \
                  [f"push_mode {args.push_mode}"] * bool(args.push_mode) + ["fused stage pipeline"] * bool(args.fused)
        if variant:  # ablation / option lines say so
            out["config"]["variant"] = ", ".join(variant)
        print(json.dumps(out), flush=True)
    ctx.close()
    if dist:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--size", default=None)
    ap.add_argument("--bin-every", type=int, default=3)
    ap.add_argument("--ref-sample", type=int, default=16_000_000)
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    # non-default decompositions / classes (the driver's runs use the defaults)
    ap.add_argument("--nradial", type=int, default=1)
    ap.add_argument("--npartdom", type=int, default=1)
    ap.add_argument("--micell", type=int, default=None)
    ap.add_argument("--mzetamax", type=int, default=None)
    ap.add_argument("--bin-mu", type=int, default=None)
    ap.add_argument("--precision", type=int, default=64, choices=[64, 32])
    # ablations of the paper's own kernel designs
    ap.add_argument("--push-mode", type=int, default=0, choices=[0, 1])
    ap.add_argument("--charge-mode", type=int, default=0, choices=[0, 1, 2])
    ap.add_argument("--fused", action="store_true", help="fused stage pipeline (one rank only)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
