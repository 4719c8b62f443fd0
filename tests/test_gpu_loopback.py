"""Decomposed-step parity on ONE GPU through the loopback transport
(gtcp_init_loopback): K contexts of this process, one host thread
and stream each, exchange every message of the decomposition -- ghost-plane
charge merge, section and ring allreduces, potential halos,
plane-split Poisson broadcasts, shift counts and payload -- with
one cudaMemcpyAsync per message.  The library code path above the transport
is the one NCCL runs (tests/dist_parity.py).  Layouts: toroidal 2 and 4,
particle replicas 2, radial windows 2 (fp32 state) and 4, toroidal x radial
2 x 2 and 2 x 4 (8 ranks), at T and at class-A geometry with 0.4-1 M markers,
class B as 8 toroidal domains of 8 planes (the 8-GPU bench layout);
plus the fixed-point scale
agreement regressions (replicas / toroidal ranks whose max|w| fall in
different binades)."""
import math

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(900)]


@pytest.fixture(scope="module")
def H():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import __graft_entry__
    __graft_entry__.build()
    import dist_harness
    return dist_harness


def _run(H, size, world, npartdom=1, nradial=1, precision=64, nparts=0, steps=2, w_scale=None, **over):
    ranks = H.LoopbackRanks(H.layout_params(size, world, npartdom, nradial, precision, **over))
    try:
        rep = H.run_parity(ranks, size, npartdom, nradial, precision, nparts, steps, w_scale=w_scale, **over)
    finally:
        ranks.close()
    return rep


CASES = [
    dict(size="T", world=2, mzetamax=8),
    dict(size="T", world=4, mzetamax=8),
    dict(size="T", world=2, npartdom=2, mzetamax=8),
    dict(size="T", world=2, nradial=2, mzetamax=8),
    dict(size="T", world=4, nradial=2, mzetamax=8),
    dict(size="T", world=4, nradial=4, mzetamax=8),               # general radial decomposition
    dict(size="A", world=8, nradial=4, nparts=400_000, steps=1, mzetamax=8),  # 2 toroidal x 4 radial
    dict(size="A", world=2, nparts=1_000_000, steps=1),
    dict(size="A", world=4, nparts=1_000_000, steps=1),
    dict(size="A", world=2, npartdom=2, nparts=1_000_000, steps=1),
    dict(size="A", world=2, nradial=2, precision=32, nparts=1_000_000, steps=1),
    dict(size="B", world=8, nparts=1_000_000, steps=1),  # the N = 8 bench layout: 8 toroidal x 8 planes
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: "-".join(f"{k}{v}" for k, v in c.items()))
def test_loopback_decomposition_parity(H, case):
    rep = _run(H, **case)
    assert rep["ok"], rep
    if case["world"] // (case.get("npartdom", 1) * case.get("nradial", 1)) > 1:
        assert rep["step0"]["movers_sent"] > 0  # the shift really moved particles


def _scale_even_ids(st):
    st["w"] = np.where(st["id"] % 2 == 0, 8.0 * st["w"], st["w"])


def _scale_first_half_torus(st):
    st["w"] = np.where(st["zeta"] < math.pi, 8.0 * st["w"], st["w"])


@pytest.mark.parametrize("layout,w_scale", [
    (dict(world=2, npartdom=2), _scale_even_ids),          # replicas in different binades (section allreduce)
    (dict(world=2), _scale_first_half_torus),              # toroidal ranks (ghost-plane merge)
    (dict(world=4, nradial=2), _scale_first_half_torus),   # toroidal x radial
], ids=["replicas", "toroidal", "toroidal-radial"])
def test_loopback_fixed_point_scale_agreement(H, layout, w_scale):
    """Ranks whose summed grids meet (ghost plane, section allreduce) must use
    one fixed-point scale: weights differing 8x between ranks put their max|w|
    in different binades; the charge must still match the oracle and every
    rank report the same fx_shift."""
    rep = _run(H, "T", mzetamax=8, steps=1, w_scale=w_scale, **layout)
    assert rep["step0"]["fx_shift_agree"] == 1, rep
    assert rep["step0"]["charge"] <= 1e-6, rep
    assert rep["ok"], rep


def test_loopback_comm_bytes_counted(H):
    """The library counts the bytes it exchanges per phase (gtcp_timings):
    the charge reduction moves at least the ghost plane, the shift at least
    the movers' 6 or 11 reals each."""
    import paper_1510_05546_b200 as G
    import synth
    ranks = H.LoopbackRanks(H.layout_params("T", 2, mzetamax=8))
    try:
        cfg = synth.config("T", mzetamax=8)
        parts = synth.load_particles(cfg, 12000, seed=3)
        P = 4
        kg = np.minimum(np.floor(parts["zeta"] * 8 / (2 * math.pi)).astype(int), 7)

        def go(r):
            c = ranks.ctx[r]
            c.set_particles({k: v[(kg // P) == r] for k, v in parts.items()})
            c.set_timing(True)
            c.timings_reset()
            c.step(1)
            return c.timings(), c.stats(), c.get_info().mgrid
        res = ranks.each(go)
    finally:
        ranks.close()
    for tm, st, mgrid in res:
        assert tm["charge_red_comm_bytes"] >= 2 * 8 * mgrid  # one int64 ghost plane per stage, at least
        assert tm["shift_comm_bytes"] >= 6 * 8 * st["movers_sent"]
        assert tm["poisson_comm_bytes"] > 0


def test_loopback_multi_hop_shift(H):
    """Multi-hop shift: 4 toroidal domains, each rank handed the
    particles of the domain two hops away; one gtcp_shift must deliver every
    particle to its owner (the movers' multi-hop flag forces the re-check
    passes that a one-hop shift skips), conserving the count and the ids."""
    import paper_1510_05546_b200 as G
    import synth
    P, K = 2, 8
    ranks = H.LoopbackRanks(H.layout_params("T", 4, mzetamax=K))
    try:
        cfg = synth.config("T", mzetamax=K)
        parts = synth.load_particles(cfg, 12000, seed=9)
        kg = np.minimum(np.floor(parts["zeta"] * K / (2 * math.pi)).astype(int), K - 1)
        owner = kg // P

        def go(r):
            c = ranks.ctx[r]
            c.set_particles({k: v[owner == (r + 2) % 4] for k, v in parts.items()})
            c.shift()
            got = c.get_particles()
            kk = np.minimum(np.floor(got["zeta"] * K / (2 * math.pi)).astype(int), K - 1)
            return got["id"], bool(np.all(kk // P == r))
        res = ranks.each(go)
    finally:
        ranks.close()
    assert all(ok for _, ok in res)
    ids = np.sort(np.concatenate([i for i, _ in res]))
    assert np.array_equal(ids, np.sort(parts["id"]))


def test_loopback_fused_pipeline_is_one_rank_only(H):
    """gtcp_set_fused is a one-rank option: a decomposed
    context rejects it (GTCP_EINVAL) and keeps stepping unfused."""
    ranks = H.LoopbackRanks(H.layout_params("T", 2, mzetamax=8))
    try:
        for c in ranks.ctx:
            with pytest.raises(Exception):
                c.set_fused(True)
            c.set_fused(False)
    finally:
        ranks.close()
