"""The C-ABI library loads, exports every symbol include/gtcp.h declares, and
its host-only calls (presets, geometry) agree with the oracle and the paper.
No compute calls (no GPU here)."""
import os
import re

import numpy as np
import pytest

import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def g():
    from paper_1510_05546_b200 import _build
    _build.build()
    import paper_1510_05546_b200 as g
    return g


def _declared():
    src = open(os.path.join(ROOT, "include", "gtcp.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gtcp_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_binding_symbols(g):
    assert _declared() == sorted(g.SYMBOLS)


def test_library_exports_every_symbol(g):
    L = g.lib()
    for name in _declared():
        assert hasattr(L, name), name
    out = os.popen(f"nm -D --defined-only {g.LIB_PATH}").read()
    for name in _declared():
        assert re.search(rf"\bT {name}\b", out), name


def test_library_is_sm100a(g):
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {g.LIB_PATH}").read()
    assert "sm_100a" in out


@pytest.mark.parametrize("size", list("TABCDabcd"))
def test_default_params_match_presets(g, size):
    p = g.gtcp_default_params(size)
    cfg = synth.config(size)
    for k in ("mpsi", "mthetamax", "mzetamax", "micell", "a0", "a1", "R0", "omega0", "q0", "q2", "rln",
              "rlt", "tau", "dt", "poisson_iters", "paranl", "w_init_amp", "vcut"):
        assert getattr(p, k) == pytest.approx(cfg[k], rel=1e-15), k


@pytest.mark.parametrize("size", list("TABCDabcd"))
def test_product_geometry_equals_oracle(g, orc, size):
    p = g.gtcp_default_params(size)
    geo = g.gtcp_geometry(p)
    og = orc.geometry(orc.make_params(synth.config(size)))
    assert geo["mgrid"] == og.mgrid
    assert np.array_equal(geo["mtheta"], og.mtheta)
    assert np.array_equal(geo["igrid"], og.igrid)
    assert np.array_equal(geo["itran"], og.itran)
    assert np.array_equal(geo["qtinv"], og.qtinv)


def test_init_rejects_bad_decomposition(g):
    p = g.gtcp_default_params("A", ntoroidal=3)  # 64 % 3 != 0
    with pytest.raises(g.GtcpError) as e:
        g.Context(p, 0, 3, nccl_id=b"\0" * 128)
    assert e.value.status in (1, 2)
