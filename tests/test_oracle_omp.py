"""The multi-core CPU baseline (oracle/gtcp_oracle_omp.c, P:330 per-thread
grid replicas summed in a fixed order) computes what the single-threaded
oracle computes: the deposit up to summation order, the push and the shift
destination bitwise (same per-particle arithmetic, split by particle range)."""
import numpy as np

import synth


def test_replica_deposit_equals_oracle(orc):
    cfg = synth.config("T")
    p = orc.make_params(cfg)
    parts = synth.load_particles(cfg, 12100, seed=1)
    a, na = orc.deposit(p, parts)
    b, nb = orc.deposit_replicas(p, parts)
    assert na == nb
    assert np.max(np.abs(a - b)) <= 1e-14 * np.sum(np.abs(parts["w"]))


def test_omp_push_and_shift_bitwise(orc):
    cfg = synth.config("T")
    p = orc.make_params(cfg)
    g = orc.geometry(p)
    parts = synth.load_particles(cfg, 5000, seed=2, w_amp=0.1)
    rng = np.random.default_rng(0)
    gp = 1e-2 * rng.standard_normal((p.mzetamax + 1, g.mgrid, 3))
    outs = []
    for fn in (orc.push, orc.push_omp):
        Xa = {k: parts[k].copy() for k in orc.ATTRS}
        Xb = {k: v.copy() for k, v in Xa.items()}
        n = fn(p, 1, Xa, Xb, parts["mu"], gp)
        outs.append((n, Xb))
    assert outs[0][0] == outs[1][0]
    for k in orc.ATTRS:
        assert np.array_equal(outs[0][1][k], outs[1][1][k])
    assert np.array_equal(orc.shift_dest(p, parts["zeta"], 1), orc.shift_dest_omp(p, parts["zeta"], 1))
