"""State snapshots in the reference's ``feklab-snapshot v1`` wire format
(format defined by feklab/solver.py:19, 179-218).

Layout (what the reference's ``save_snapshot`` / ``load_snapshot`` exchange):

    b"feklab-snapshot v1\\n"
    one JSON line, keys sorted:
        {"arrays": {name: {"offset": byte offset in the payload,
                           "shape": [...]}},
         "dtype": "<f8",
         "mesh": {"nx", "ny", "nz", "extents"}}          (only with a mesh)
    payload: the little-endian float64 arrays u, p[, eta][, vertices]
             back to back in that order

This implementation is built for device-resident states: arrays are
streamed to the file in bounded chunks (a CUDA tensor is staged through one
reused pinned host buffer, so a multi-GB state never needs a full host
copy), and loading can map the payload lazily (``mmap=True``) or land the
arrays straight on a CUDA device.  Files are byte-identical to the
reference's for the same state (tests/test_snapshot.py checks a file the
reference itself wrote).
"""

from __future__ import annotations

import json
import os

import numpy as np

MAGIC = b"feklab-snapshot v1\n"
DTYPE = np.dtype("<f8")
_CHUNK = 32 << 20  # bytes per streamed piece


def _fields(state, mesh):
    """(name, array-like) in the reference's payload order."""
    items = [("u", state.u), ("p", state.p)]
    if getattr(state, "eta", None) is not None:
        items.append(("eta", state.eta))
    if mesh is not None:
        items.append(("vertices", mesh.vertices))
    return items


def _shape(a) -> list[int]:
    return [int(s) for s in a.shape]


def _nbytes(a) -> int:
    return int(np.prod(_shape(a), dtype=np.int64)) * DTYPE.itemsize


def _header_line(items, mesh) -> bytes:
    arrays, pos = {}, 0
    for name, a in items:
        arrays[name] = {"offset": pos, "shape": _shape(a)}
        pos += _nbytes(a)
    head = {"arrays": arrays, "dtype": DTYPE.str}
    if mesh is not None:
        head["mesh"] = {"extents": [float(e) for e in mesh.extents],
                        "nx": int(mesh.nx), "ny": int(mesh.ny), "nz": int(mesh.nz)}
    return json.dumps(head, sort_keys=True).encode() + b"\n"


class _Stager:
    """One pinned host buffer reused for every device -> file piece."""

    def __init__(self):
        self.buf = None

    def pieces(self, t):
        import torch

        flat = t.detach().reshape(-1)
        if flat.dtype != torch.float64:
            flat = flat.to(torch.float64)
        step = _CHUNK // DTYPE.itemsize
        if self.buf is None or self.buf.numel() < min(step, flat.numel()):
            self.buf = torch.empty(min(step, max(1, flat.numel())), dtype=torch.float64,
                                   pin_memory=True)
        for s in range(0, flat.numel(), step):
            n = min(step, flat.numel() - s)
            self.buf[:n].copy_(flat[s:s + n])  # synchronous D2H into pinned memory
            yield self.buf[:n].numpy().astype(DTYPE, copy=False).tobytes()


def _host_pieces(a):
    flat = np.ascontiguousarray(np.asarray(a), dtype=DTYPE).reshape(-1)
    step = _CHUNK // DTYPE.itemsize
    for s in range(0, flat.size, step):
        yield memoryview(flat[s:s + step]).cast("B")


def save_snapshot(path, state, mesh=None) -> None:
    """Write ``state`` (``.u``, ``.p``, optional ``.eta``; NumPy arrays or
    torch tensors on any device) and optionally the mesh vertices."""
    items = _fields(state, mesh)
    stager = _Stager()
    with open(path, "wb") as fh:
        fh.write(MAGIC)
        fh.write(_header_line(items, mesh))
        for _, a in items:
            is_cuda = getattr(a, "is_cuda", False)
            for piece in (stager.pieces(a) if is_cuda else
                          _host_pieces(a.detach().cpu().numpy() if hasattr(a, "detach") else a)):
                fh.write(piece)


def read_header(path) -> tuple[dict, int]:
    """(header dict, byte offset of the payload)."""
    with open(path, "rb") as fh:
        if fh.readline() != MAGIC:
            fh.seek(0)
            got = fh.readline().decode(errors="replace").strip()
            raise ValueError(f"not a snapshot file (magic {got!r})")
        head = json.loads(fh.readline().decode())
        return head, fh.tell()


def load_snapshot(path, mmap: bool = False, device=None) -> dict:
    """{name: array, ..., "mesh_meta": {...}} like the reference's
    ``load_snapshot``.  ``mmap=True`` returns read-only memory-mapped views;
    ``device`` (e.g. "cuda") returns torch tensors on that device."""
    head, base = read_header(path)
    dt = np.dtype(head["dtype"])
    size = os.path.getsize(path)
    out = {}
    for name, meta in head["arrays"].items():
        shape = tuple(meta["shape"])
        count = int(np.prod(shape, dtype=np.int64)) if shape else 1
        start = base + int(meta["offset"])
        if start + count * dt.itemsize > size:
            raise ValueError(f"snapshot array {name!r} runs past the end of the file")
        if mmap:
            arr = np.memmap(path, dtype=dt, mode="r", offset=start, shape=shape or (1,))
        else:
            arr = np.fromfile(path, dtype=dt, count=count, offset=start).reshape(shape)
        if device is not None:
            import torch

            arr = torch.as_tensor(np.ascontiguousarray(arr, dtype=np.float64), device=device)
        out[name] = arr
    if "mesh" in head:
        out["mesh_meta"] = head["mesh"]
    return out
