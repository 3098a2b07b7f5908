"""ctypes binding of libfk_b200.so (include/fk.h).

This is the same binding a maintainer would add to feklab.
There is no CPU fallback: if the library is missing the import of the
operator module fails loudly.
"""

from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libfk_b200.so")

FK_OK = 0
FK_EINVAL = -1
FK_ECUDA = -2
FK_ENCCL = -3
FK_ENOMEM = -4
FK_EUNSUPPORTED = -5

FK_KIND_MASS = 1
FK_KIND_DIFFUSION = 3

FK_VARIANT_AUTO = 0
FK_VARIANT_DFMA = 1
FK_VARIANT_DMMA = 2

FK_VARIANT_EO = 3
FK_VARIANT_MF = 4

FK_TRANSPORT_NCCL = 1
FK_TRANSPORT_P2P = 2
FK_MAX_RANKS = 16
FK_IPC_HANDLE_BYTES = 64
TRANSPORTS = {"nccl": FK_TRANSPORT_NCCL, "p2p": FK_TRANSPORT_P2P}

VARIANTS = {"auto": FK_VARIANT_AUTO, "dfma": FK_VARIANT_DFMA, "dmma": FK_VARIANT_DMMA,
            "eo": FK_VARIANT_EO, "mf": FK_VARIANT_MF}
VARIANT_NAMES = {v: k for k, v in VARIANTS.items()}

#: every symbol include/fk.h declares (checked by tests/test_cabi.py)
EXPORTS = (
    "fk_version", "fk_last_error", "fk_op_create", "fk_op_setup", "fk_op_destroy",
    "fk_op_get_info", "fk_op_set_variant", "fk_op_set_config", "fk_op_restriction",
    "fk_op_pa_data",
    "fk_op_apply", "fk_op_apply_host", "fk_op_apply_local", "fk_op_diagonal",
    "fk_op_set_essential",
    "fk_cg_prepare", "fk_cg_solve", "fk_dot", "fk_comm_unique_id", "fk_comm_create",
    "fk_comm_create_p2p", "fk_comm_connect_p2p", "fk_comm_create_loopback", "fk_comm_query",
    "fk_comm_destroy",
    "fk_op_time_apply",
    "fk_mix_create", "fk_mix_setup", "fk_mix_destroy", "fk_mix_get_info", "fk_mix_apply",
    "fk_mix_fused_normal", "fk_mix_mass_inverse", "fk_mix_rk4", "fk_mix_rk4_forced",
    "fk_mix_bottom_load", "fk_mix_lumped",
    "fk_mix_restriction", "fk_mix_time_apply",
)


class FkOpDesc(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int),
        ("p", ctypes.c_int),
        ("q", ctypes.c_int),
        ("nx", ctypes.c_int),
        ("ny", ctypes.c_int),
        ("nz_local", ctypes.c_int),
        ("z0_layer", ctypes.c_int),
        ("nz_global", ctypes.c_int),
        ("jac_diag", ctypes.c_double * 3),
        ("jac_det", ctypes.c_double),
        ("B", ctypes.POINTER(ctypes.c_double)),
        ("G", ctypes.POINTER(ctypes.c_double)),
        ("w", ctypes.POINTER(ctypes.c_double)),
        ("gather_ids", ctypes.POINTER(ctypes.c_int64)),
        ("dirichlet", ctypes.c_int),
        ("variant", ctypes.c_int),
        ("device", ctypes.c_int),
        ("stream", ctypes.c_void_p),
        ("comm", ctypes.c_void_p),
        ("deterministic", ctypes.c_int),
    ]


class FkOpInfo(ctypes.Structure):
    _fields_ = [
        ("ndof_local", ctypes.c_int64),
        ("nel_local", ctypes.c_int64),
        ("dof_offset", ctypes.c_int64),
        ("ndof_global", ctypes.c_int64),
        ("pa_bytes", ctypes.c_int64),
        ("variant", ctypes.c_int),
        ("elems_per_block", ctypes.c_int),
        ("threads_per_block", ctypes.c_int),
        ("blocks", ctypes.c_int),
        ("cfg", ctypes.c_int),
    ]


class FkMixDesc(ctypes.Structure):
    _fields_ = [
        ("order_p", ctypes.c_int),
        ("order_u", ctypes.c_int),
        ("num_quad_1d", ctypes.c_int),
        ("nx", ctypes.c_int),
        ("ny", ctypes.c_int),
        ("nz", ctypes.c_int),
        ("jac_diag", ctypes.c_double * 3),
        ("jac_det", ctypes.c_double),
        ("Bp", ctypes.POINTER(ctypes.c_double)),
        ("Gp", ctypes.POINTER(ctypes.c_double)),
        ("Bu", ctypes.POINTER(ctypes.c_double)),
        ("w", ctypes.POINTER(ctypes.c_double)),
        ("rho", ctypes.POINTER(ctypes.c_double)),
        ("bulk", ctypes.POINTER(ctypes.c_double)),
        ("rho_scalar", ctypes.c_double),
        ("bulk_scalar", ctypes.c_double),
        ("coupling_scale", ctypes.c_double),
        ("matrix_free", ctypes.c_int),
        ("device", ctypes.c_int),
        ("stream", ctypes.c_void_p),
        ("absorbing", ctypes.c_int),
        ("surface_gravity", ctypes.c_double),
    ]


class FkMixInfo(ctypes.Structure):
    _fields_ = [
        ("nel", ctypes.c_int64),
        ("ndof_p", ctypes.c_int64),
        ("ndof_u", ctypes.c_int64),
        ("pa_bytes", ctypes.c_int64),
        ("elems_per_block", ctypes.c_int),
        ("threads_per_block", ctypes.c_int),
        ("blocks", ctypes.c_int),
        ("smem_bytes", ctypes.c_int64),
    ]


_lib = None


def load(path: str | None = None) -> ctypes.CDLL:
    """Load (once) and type the C-ABI.  Raises if the library was not built."""
    global _lib
    if _lib is not None:
        return _lib
    # FK_LIB_PATH: an alternative build of the same library (A/B tooling,
    # tools/build_variant.py); never set on the product path
    path = path or os.environ.get("FK_LIB_PATH") or LIB_PATH
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build it with `python -m paper_2603_09038_b200.build` "
            "(there is no CPU fallback)")
    if "FK_NCCL_LIBRARY" not in os.environ:
        try:
            import nvidia.nccl  # type: ignore

            for p in nvidia.nccl.__path__:
                cand = os.path.join(p, "lib", "libnccl.so.2")
                if os.path.exists(cand):
                    os.environ["FK_NCCL_LIBRARY"] = cand
                    break
        except Exception:
            pass
    lib = ctypes.CDLL(path)
    vp, i, d, i64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_double, ctypes.c_int64
    pd = ctypes.POINTER(ctypes.c_double)
    sig = {
        "fk_version": (i, []),
        "fk_last_error": (ctypes.c_char_p, []),
        "fk_op_create": (i, [ctypes.POINTER(vp), ctypes.POINTER(FkOpDesc)]),
        "fk_op_setup": (i, [vp]),
        "fk_op_destroy": (i, [vp]),
        "fk_op_get_info": (i, [vp, ctypes.POINTER(FkOpInfo)]),
        "fk_op_set_variant": (i, [vp, i]),
        "fk_op_set_config": (i, [vp, i, i]),
        "fk_op_restriction": (i, [vp, ctypes.POINTER(i64)]),
        "fk_op_pa_data": (i, [vp, pd]),
        "fk_op_apply": (i, [vp, vp, vp]),
        "fk_op_apply_host": (i, [vp, vp, vp]),
        "fk_op_apply_local": (i, [vp, vp, vp]),
        "fk_op_diagonal": (i, [vp, vp]),
        "fk_op_set_essential": (i, [vp, vp, d]),
        "fk_cg_prepare": (i, [vp, i]),
        "fk_cg_solve": (i, [vp, vp, vp, i, d, pd, ctypes.POINTER(i)]),
        "fk_dot": (i, [vp, vp, vp, pd]),
        "fk_comm_unique_id": (i, [vp]),
        "fk_comm_create": (i, [ctypes.POINTER(vp), vp, i, i, i]),
        "fk_comm_create_p2p": (i, [ctypes.POINTER(vp), i, i, i, i64, vp]),
        "fk_comm_connect_p2p": (i, [vp, vp]),
        "fk_comm_create_loopback": (i, [ctypes.POINTER(vp), i, ctypes.POINTER(i), i64]),
        "fk_comm_query": (i, [vp, ctypes.POINTER(i), ctypes.POINTER(i), ctypes.POINTER(i)]),
        "fk_comm_destroy": (i, [vp]),
        "fk_op_time_apply": (i, [vp, vp, vp, i, vp, ctypes.c_size_t, pd, pd]),
        "fk_mix_create": (i, [ctypes.POINTER(vp), ctypes.POINTER(FkMixDesc)]),
        "fk_mix_setup": (i, [vp]),
        "fk_mix_destroy": (i, [vp]),
        "fk_mix_get_info": (i, [vp, ctypes.POINTER(FkMixInfo)]),
        "fk_mix_apply": (i, [vp, vp, vp, vp, vp]),
        "fk_mix_fused_normal": (i, [vp, vp, vp]),
        "fk_mix_mass_inverse": (i, [vp, vp, vp, vp, vp]),
        "fk_mix_rk4": (i, [vp, vp, vp, d, i]),
        "fk_mix_rk4_forced": (i, [vp, vp, vp, d, vp, vp, vp]),
        "fk_mix_bottom_load": (i, [vp, vp, vp]),
        "fk_mix_lumped": (i, [vp, vp, vp]),
        "fk_mix_restriction": (i, [vp, ctypes.POINTER(i64)]),
        "fk_mix_time_apply": (i, [vp, vp, vp, vp, vp, i, pd, pd]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


class FkError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"fk error {code}: {msg}")
        self.code = code


def check(rc: int) -> None:
    if rc == FK_OK:
        return
    msg = _lib.fk_last_error().decode(errors="replace") if _lib else "?"
    if rc == FK_EINVAL:
        raise ValueError(msg)
    if rc == FK_EUNSUPPORTED:
        raise NotImplementedError(msg)
    if rc == FK_ENOMEM:
        raise MemoryError(msg)
    raise FkError(rc, msg)
