"""State snapshot files in the reference's wire format.

``feklab-snapshot v1`` (feklab/solver.py:19, 179-218): a magic line, one JSON
header line (``{"arrays": {name: {"offset", "shape"}}, "dtype": "<f8",
"mesh": {...}}``, keys sorted), then the little-endian float64 payloads of
``u``, ``p`` (and ``eta``, ``vertices``) back to back.  Files written here are
byte-identical to the reference's ``save_snapshot`` for the same state and
load with its ``load_snapshot``, so device states can be exchanged with the
CPU path.  CUDA tensors are copied to the host.
"""

from __future__ import annotations

import json

import numpy as np

SNAP_MAGIC = "feklab-snapshot v1"


def _host(a) -> np.ndarray:
    if isinstance(a, np.ndarray):
        return a
    return a.detach().cpu().numpy()


def save_snapshot(path, state, mesh=None) -> None:
    """Write ``state`` (``.u``, ``.p``, optional ``.eta``) like
    feklab.solver.save_snapshot (solver.py:179-198)."""
    arrays = {"u": _host(state.u), "p": _host(state.p)}
    eta = getattr(state, "eta", None)
    if eta is not None:
        arrays["eta"] = _host(eta)
    if mesh is not None:
        arrays["vertices"] = _host(mesh.vertices)
    header: dict = {"arrays": {}, "dtype": "<f8"}
    if mesh is not None:
        header["mesh"] = {"nx": mesh.nx, "ny": mesh.ny, "nz": mesh.nz,
                          "extents": tuple(float(x) for x in mesh.extents)}
    offset = 0
    blobs = []
    for name, arr in arrays.items():
        a = np.ascontiguousarray(arr, dtype="<f8")
        header["arrays"][name] = {"shape": list(a.shape), "offset": offset}
        blobs.append(a.tobytes())
        offset += len(blobs[-1])
    with open(path, "wb") as fh:
        fh.write(SNAP_MAGIC.encode() + b"\n")
        fh.write(json.dumps(header, sort_keys=True).encode() + b"\n")
        for blob in blobs:
            fh.write(blob)


def load_snapshot(path) -> dict:
    """Read a snapshot (feklab.solver.load_snapshot, solver.py:201-218):
    {name: ndarray, ..., "mesh_meta": {...}}."""
    with open(path, "rb") as fh:
        magic = fh.readline().decode().strip()
        if magic != SNAP_MAGIC:
            raise ValueError(f"not a snapshot file (magic {magic!r})")
        header = json.loads(fh.readline().decode())
        payload = fh.read()
    out = {}
    for name, meta in header["arrays"].items():
        shape = tuple(meta["shape"])
        count = int(np.prod(shape)) if shape else 1
        arr = np.frombuffer(payload, dtype=header["dtype"], count=count, offset=meta["offset"])
        out[name] = arr.reshape(shape).copy()
    if "mesh" in header:
        out["mesh_meta"] = header["mesh"]
    return out
