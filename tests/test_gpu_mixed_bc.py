"""Acoustic-gravity block operator: boundary terms, forcing and counters on
the B200 path against golden vectors of the real reference
(tests/golden/make_golden_mixed_bc.py; operator.py:268-276, 357-358,
432-470, 506-531, counters of :280-286)."""

import os

import numpy as np
import pytest

from _util import PARITY_TOL, normwise
from paper_2603_09038_b200 import Counters, MixedOperator, MixedState, build_mesh, rk4_step

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

G = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden_mixed_bc.npz"))
NAMES = ["b222", "b322_p2", "b232_p3cs", "b333_p6"]


def profile(x, y):
    return np.sin(np.pi * x) * np.cos(0.5 * y) + 0.25 * x * y


def make(name, **kw):
    m = G[f"{name}_meta"]
    n = tuple(int(v) for v in m[:3])
    mesh = build_mesh(*n, extents=tuple(float(v) for v in m[3:6]))
    return MixedOperator(mesh, int(m[6]), int(m[7]), int(m[8]), rho=G[f"{name}_rho"],
                         bulk_modulus=G[f"{name}_bulk"], coupling_scale=float(m[11]), **kw), float(m[12])


@pytest.mark.parametrize("name", NAMES)
@pytest.mark.parametrize("strategy", ["FusedPA", "FusedMF"])
def test_absorbing_apply(name, strategy):
    op, _ = make(name, absorbing=True, strategy=strategy)
    r = op.apply(MixedState(G[f"{name}_u"], G[f"{name}_p"]))
    assert normwise(r.u, G[f"{name}_absorb_out_u"]) <= PARITY_TOL
    assert normwise(r.p, G[f"{name}_absorb_out_p"]) <= PARITY_TOL


@pytest.mark.parametrize("name", NAMES)
def test_surface_gravity_mass_and_height(name):
    op, g = make(name, surface_gravity=None)
    opg, g = make(name, surface_gravity=g)
    _, lp = opg.lumped()
    assert normwise(lp, G[f"{name}_surf_lump_p"]) <= 1e-14
    s = MixedState(G[f"{name}_u"], G[f"{name}_p"])
    assert normwise(opg.apply_mass_inverse(s).p, G[f"{name}_surf_minv_p"]) <= 1e-14
    assert np.array_equal(opg.surface_height(s), G[f"{name}_surf_height"])
    with pytest.raises(ValueError, match="without surface gravity"):
        op.surface_height(s)


@pytest.mark.parametrize("name", NAMES)
def test_bottom_face_load(name):
    op, _ = make(name)
    assert normwise(op.bottom_face_load(profile), G[f"{name}_bottom_load"]) <= PARITY_TOL


@pytest.mark.parametrize("name", NAMES)
def test_forced_rk4_with_boundary_terms(name):
    op, g = make(name, absorbing=True, surface_gravity=None)
    op, g = make(name, absorbing=True, surface_gravity=g)
    u0, p0 = G[f"{name}_u"], G[f"{name}_p"]

    def forcing(t):
        return MixedState(np.sin(3.0 * t) * u0[::-1].copy(),
                          np.cos(2.0 * t) * np.linspace(-1.0, 1.0, op.num_p))

    st = MixedState(u0.copy(), p0.copy())
    for k in range(2):
        st = rk4_step(st, 2e-3, op, forcing=forcing, t=0.25 + k * 2e-3, step_index=k)
    assert normwise(st.u, G[f"{name}_rk4f_u"]) <= PARITY_TOL
    assert normwise(st.p, G[f"{name}_rk4f_p"]) <= PARITY_TOL
    assert op.counters.operator_applies == 8


@pytest.mark.parametrize("name", NAMES)
def test_counters_match_reference(name):
    s = MixedState(G[f"{name}_u"], G[f"{name}_p"])
    for strat in ("PA", "FusedPA", "MF", "FusedMF"):
        c = Counters()
        op, _ = make(name, strategy=strat, counters=c)
        op.apply(s)
        a = (c.operator_applies, c.flops, c.d_reads)
        c.operator_applies = c.flops = c.d_reads = 0
        op.apply_fused_normal(s.u)
        assert a + (c.operator_applies, c.flops, c.d_reads) == tuple(G[f"{name}_counters_{strat}"])


def test_reference_d_read_semantics():
    """feklab tests/test_operator.py:271-289 against MixedOperator."""
    mesh = build_mesh(2, 2, 2)
    ops = {s: MixedOperator(mesh, strategy=s) for s in ("PA", "FusedPA", "MF")}
    rng = np.random.default_rng(3)
    st = ops["PA"].zero_state()
    st = MixedState(rng.standard_normal(st.u.shape), rng.standard_normal(st.p.shape))
    for o in ops.values():
        o.counters.reset() if hasattr(o.counters, "reset") else None
        o.apply(st)
    assert ops["PA"].counters.d_reads == 2 * ops["FusedPA"].counters.d_reads > 0
    assert ops["MF"].counters.d_reads == 0


def test_bad_gravity():
    with pytest.raises(ValueError, match="positive"):
        MixedOperator(build_mesh(2, 2, 2), surface_gravity=-1.0)
