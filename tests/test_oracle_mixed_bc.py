"""Oracle restatement of the block operator's boundary terms, forcing and
counters against golden vectors produced by the real reference
(tests/golden/make_golden_mixed_bc.py): bit-exact where the reference's
arithmetic is elementwise NumPy."""

import os

import numpy as np
import pytest

from oracle.mixed import MixedProblem

G = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden_mixed_bc.npz"))
NAMES = ["b222", "b322_p2", "b232_p3cs", "b333_p6"]


def profile(x, y):
    return np.sin(np.pi * x) * np.cos(0.5 * y) + 0.25 * x * y


def problem(name):
    m = G[f"{name}_meta"]
    n = tuple(int(v) for v in m[:3])
    M = MixedProblem(*n, int(m[6]), int(m[7]), int(m[8]), extents=tuple(m[3:6]),
                     rho=G[f"{name}_rho"], bulk=G[f"{name}_bulk"], coupling_scale=m[11])
    return M, float(m[12])


def forcing_for(M, u):
    def f(t):
        return np.sin(3.0 * t) * u[::-1].copy(), np.cos(2.0 * t) * np.linspace(-1.0, 1.0, M.ndof_p)
    return f


@pytest.mark.parametrize("name", NAMES)
def test_boundary_terms_bit_exact(name):
    M, g = problem(name)
    u, p = G[f"{name}_u"], G[f"{name}_p"]
    ru, rp = M.apply_absorbing(u, p)
    assert np.array_equal(ru, G[f"{name}_absorb_out_u"]) and np.array_equal(rp, G[f"{name}_absorb_out_p"])
    assert np.array_equal(M.surface_lump_p(g), G[f"{name}_surf_lump_p"])
    assert np.array_equal(M.surface_height(p, g), G[f"{name}_surf_height"])
    assert np.array_equal(M.bottom_face_load(profile), G[f"{name}_bottom_load"])
    lp = M.surface_lump_p(g)
    assert np.array_equal(p / lp, G[f"{name}_surf_minv_p"])


@pytest.mark.parametrize("name", NAMES)
def test_forced_rk4_and_counters(name):
    M, g = problem(name)
    u, p = G[f"{name}_u"], G[f"{name}_p"]
    # the golden RK4 runs on an operator with absorbing faces + surface gravity
    M.lump_p = M.surface_lump_p(g)
    M.apply = M.apply_absorbing
    f = forcing_for(M, u)
    uu, pp = u, p
    for k in range(2):
        uu, pp = M.rk4_step(uu, pp, 2e-3, forcing=f, t=0.25 + k * 2e-3)
    su = np.max(np.abs(G[f"{name}_rk4f_u"]))
    assert np.max(np.abs(uu - G[f"{name}_rk4f_u"])) <= 1e-14 * su
    assert np.max(np.abs(pp - G[f"{name}_rk4f_p"])) <= 1e-14 * np.max(np.abs(G[f"{name}_rk4f_p"]))
    for s in ("PA", "FusedPA", "MF", "FusedMF"):
        c = G[f"{name}_counters_{s}"]
        assert M.counts(s) == tuple(c[:3]) and M.counts(s, normal=True) == tuple(c[3:])
