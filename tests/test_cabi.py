"""The C-ABI library loads and exports every symbol include/fk.h declares.

CPU-only: no compute calls; descriptor validation runs before any CUDA call,
so argument errors are checked here too.
"""

import ctypes
import os
import re

import numpy as np
import pytest

from paper_2603_09038_b200 import _lib

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "fk.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fk_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    decl = declared_functions()
    assert len(decl) >= 15
    for name in decl:
        assert hasattr(lib, name), name
    assert sorted(decl) == sorted(_lib.EXPORTS)


def test_version():
    assert _lib.load().fk_version() == 2


def _desc(**kw):
    B = np.zeros((6, 5))
    d = _lib.FkOpDesc()
    d.kind, d.p, d.q = 3, 4, 6
    d.nx = d.ny = d.nz_local = d.nz_global = 2
    d.z0_layer = 0
    for s in range(3):
        d.jac_diag[s] = 0.25
    d.jac_det = 0.25 ** 3
    dp = ctypes.POINTER(ctypes.c_double)
    d._keep = B
    d.B = d.G = d.w = B.ctypes.data_as(dp)
    for k, v in kw.items():
        setattr(d, k, v)
    return d


@pytest.mark.parametrize("kw,code,needle", [
    (dict(kind=2), _lib.FK_EINVAL, "kind"),
    (dict(p=9, q=11), _lib.FK_EUNSUPPORTED, "order"),
    (dict(q=4), _lib.FK_EUNSUPPORTED, "num_quad_1d"),
    (dict(nz_local=3), _lib.FK_EINVAL, "do not match"),
    (dict(jac_det=0.0), _lib.FK_EINVAL, "Jacobian"),
    # maximum size: int32 dof ids (the device E-restriction) cap a rank at < 2^31 dofs
    (dict(nx=2300, ny=2300, nz_local=60, nz_global=60), _lib.FK_EINVAL, "too large"),
    (dict(variant=7), _lib.FK_EINVAL, "variant"),
])
def test_descriptor_validation(kw, code, needle):
    lib = _lib.load()
    h = ctypes.c_void_p()
    rc = lib.fk_op_create(ctypes.byref(h), ctypes.byref(_desc(**kw)))
    assert rc == code
    assert needle in lib.fk_last_error().decode()
    assert not h.value


def test_null_arguments():
    lib = _lib.load()
    assert lib.fk_op_apply(None, None, None) == _lib.FK_EINVAL
    assert lib.fk_op_setup(None) == _lib.FK_EINVAL
    assert lib.fk_op_destroy(None) == _lib.FK_OK


def test_check_maps_codes_to_python_errors():
    _lib.load()
    with pytest.raises(ValueError):
        _lib.check(_lib.FK_EINVAL)
    with pytest.raises(NotImplementedError):
        _lib.check(_lib.FK_EUNSUPPORTED)
    with pytest.raises(RuntimeError):
        _lib.check(_lib.FK_ECUDA)


def test_no_cpu_fallback_in_product():
    # the product package never imports the oracle
    root = os.path.join(os.path.dirname(HEADER), "..", "paper_2603_09038_b200")
    for dirpath, _, files in os.walk(root):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f


def test_bench_module_imports():
    """bench.py (the driver's entry point) parses and its CLI builds."""
    import importlib.util
    import os
    import sys

    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "bench.py")
    spec = importlib.util.spec_from_file_location("bench_under_test", path)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    argv = sys.argv
    try:
        sys.argv = ["bench.py", "--gpus", "1", "--steps", "3", "--warmup", "3"]
        a = mod.parse()
    finally:
        sys.argv = argv
    assert a.steps == 3 and a.impl == "ours"


def _mix_desc(**kw):
    d = _lib.FkMixDesc()
    d.order_p, d.order_u, d.num_quad_1d = 4, 3, 5
    d.nx = d.ny = d.nz = 2
    for s in range(3):
        d.jac_diag[s] = 0.25
    d.jac_det = 0.25 ** 3
    T = np.zeros((5, 5))
    dp = ctypes.POINTER(ctypes.c_double)
    d._keep = T
    d.Bp = d.Gp = d.Bu = d.w = T.ctypes.data_as(dp)
    d.rho_scalar = d.bulk_scalar = 1.0
    d.coupling_scale = 1.0
    for k, v in kw.items():
        setattr(d, k, v)
    return d


@pytest.mark.parametrize("kw,code,needle", [
    (dict(order_p=1, order_u=0, num_quad_1d=2), _lib.FK_EUNSUPPORTED, "order_p"),
    (dict(order_u=2), _lib.FK_EUNSUPPORTED, "order_u"),
    (dict(num_quad_1d=6), _lib.FK_EUNSUPPORTED, "q"),
    (dict(nz=0), _lib.FK_EINVAL, "do not match"),
    (dict(jac_det=0.0), _lib.FK_EINVAL, "Jacobian"),
    (dict(rho_scalar=-1.0), _lib.FK_EINVAL, "positive"),
])
def test_mix_create_validates(kw, code, needle):
    """fk_mix_create (acoustic-gravity operator) validates the descriptor on the
    host, with the reference's wording where it has one (operator.py:129-130,
    160-161)."""
    lib = _lib.load()
    h = ctypes.c_void_p()
    d = _mix_desc(**kw)
    rc = lib.fk_mix_create(ctypes.byref(h), ctypes.byref(d))
    assert rc == code
    assert needle in lib.fk_last_error().decode()
