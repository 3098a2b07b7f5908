"""FP64 m8n8k4 tile maps in the reference's ``feklab-mapping v1`` text format
(the format and its semantics are defined by
feklab/mma.py: GemmShape :36-67, IndexMapping :151-207, the identity /
column-permuted / hand-tuned maps :210-249, the file codec :385-474, and the
seven shipped ``mappings/*.map`` files).

A map assigns every slot of the instruction tiles a problem index: per warp
an 8-row map ``f_m[w]``, one column map ``f_n`` (8 per n-tile) and one
reduction map ``f_k`` (4 per k-tile) shared by the warps; ``PAD`` (-1)
slots read zero and are dropped.  The text form lists, warp-major, every
slot triple ``w mi ni ki -> m n k`` (or ``-> PAD``).

Here the codec is vectorised (NumPy index grids instead of nested loops,
one regular expression pass for parsing) so the large maps of the higher
orders round-trip quickly, and ``lane_tables`` turns a map into the
per-lane operand/accumulator coordinates of ``mma.sync.m8n8k4.f64``
(lane L: A(L/4, L%4), B(L%4, L/4), C(L/4, 2(L%4)+{0,1}); mma.py:70-120)
that a DMMA kernel addresses shared memory with.  Output is byte-identical
to the reference's files (tests/test_mapping.py).
"""
from __future__ import annotations

import re
from dataclasses import dataclass, field

import numpy as np

PAD = -1
INSTR_M, INSTR_N, INSTR_K = 8, 8, 4
_TAG = "feklab-mapping"
_VERSION = "v1"


class CoverageError(ValueError):
    """A map double-covers or misses problem indices."""


class MappingFormatError(ValueError):
    """Text that is not a well-formed map file."""


@dataclass(frozen=True)
class GemmShape:
    """Problem GEMM (m x k) @ (k x n); text form ``MxNxK``."""

    m: int
    n: int
    k: int

    def __post_init__(self):
        if min(self.m, self.n, self.k) < 1:
            raise ValueError(f"all GEMM dimensions must be >= 1, got {self}")

    @classmethod
    def parse(cls, text: str) -> "GemmShape":
        nums = re.split(r"[xX/]", text.strip())
        if len(nums) != 3:
            raise ValueError(f"expected MxNxK, got {text!r}")
        return cls(*(int(v) for v in nums))

    def __str__(self) -> str:
        return "x".join(str(v) for v in (self.m, self.n, self.k))

    def tiles(self, extent: int, width: int) -> int:
        return -(-extent // width)

    m_tiles = property(lambda self: self.tiles(self.m, INSTR_M))
    n_tiles = property(lambda self: self.tiles(self.n, INSTR_N))
    k_tiles = property(lambda self: self.tiles(self.k, INSTR_K))


def _axis_errors(name: str, slots: np.ndarray, extent: int) -> str | None:
    live = slots[slots != PAD]
    stray = live[(live < 0) | (live >= extent)]
    if stray.size:
        return f"f_{name} maps outside [0, {extent}): {sorted(set(stray.tolist()))}"
    hits = np.bincount(live, minlength=extent)
    if np.any(hits != 1):
        return (f"f_{name} coverage broken: duplicated {np.flatnonzero(hits > 1).tolist()}, "
                f"missing {np.flatnonzero(hits == 0).tolist()}")
    return None


@dataclass
class IndexMapping:
    """Slot maps of one tiled GEMM: ``f_m`` (warps, 8), ``f_n`` (8 ntiles,),
    ``f_k`` (4 ktiles,), int64 with PAD = -1."""

    shape: GemmShape
    f_m: np.ndarray
    f_n: np.ndarray
    f_k: np.ndarray
    _ok: bool = field(default=False, repr=False, compare=False)

    def __post_init__(self):
        self.f_m, self.f_n, self.f_k = (np.asarray(a, dtype=np.int64)
                                        for a in (self.f_m, self.f_n, self.f_k))
        checks = ((self.f_m.ndim == 2 and self.f_m.shape[-1] == INSTR_M,
                   f"f_m must be (warps, 8), got {self.f_m.shape}"),
                  (self.f_n.ndim == 1 and self.f_n.size % INSTR_N == 0,
                   f"f_n must span a multiple of 8 slots, got {self.f_n.shape}"),
                  (self.f_k.ndim == 1 and self.f_k.size % INSTR_K == 0,
                   f"f_k must span a multiple of 4 slots, got {self.f_k.shape}"))
        for ok, msg in checks:
            if not ok:
                raise CoverageError(msg)

    num_warps = property(lambda self: int(self.f_m.shape[0]))
    n_tiles = property(lambda self: self.f_n.size // INSTR_N)
    k_tiles = property(lambda self: self.f_k.size // INSTR_K)

    def validate_coverage(self) -> None:
        """Every problem index on m, n and k comes from exactly one slot."""
        for name, slots, extent in (("m", self.f_m.ravel(), self.shape.m),
                                    ("n", self.f_n, self.shape.n),
                                    ("k", self.f_k, self.shape.k)):
            err = _axis_errors(name, slots, extent)
            if err:
                raise CoverageError(err)


def _iota(slots: int, extent: int) -> np.ndarray:
    v = np.arange(slots, dtype=np.int64)
    return np.where(v < extent, v, PAD)


def identity_mapping(shape: GemmShape) -> IndexMapping:
    """Warp w owns rows 8w..8w+7; identity column and reduction slots."""
    return IndexMapping(shape, _iota(shape.m_tiles * INSTR_M, shape.m).reshape(-1, INSTR_M),
                        _iota(shape.n_tiles * INSTR_N, shape.n), _iota(shape.k_tiles * INSTR_K, shape.k))


def column_permuted_mapping(shape: GemmShape, n_perm) -> IndexMapping:
    """The identity map with its eight column slots reordered by ``n_perm``."""
    perm = np.asarray([int(v) for v in n_perm], dtype=np.int64)
    if perm.size != INSTR_N or not np.array_equal(np.sort(perm), np.arange(INSTR_N)):
        raise ValueError(f"n_perm must permute 0..7, got {perm.tolist()}")
    base = identity_mapping(shape)
    base.f_n = np.where(perm < shape.n, perm, PAD)
    return base


HAND_TUNED_COLUMN_PERM = (0, 2, 1, 3, 4, 5, 6, 7)


def hand_tuned_mapping_25x5x4() -> IndexMapping:
    """Four row-blocked warps, column slots 1 and 2 exchanged (mma.py:238-249)."""
    return column_permuted_mapping(GemmShape(25, 5, 4), HAND_TUNED_COLUMN_PERM)


# -- codec ----------------------------------------------------------------------------


def format_mapping(mp: IndexMapping) -> str:
    """The text file: header, then one line per slot triple, warp-major,
    then m slot, n slot, k slot."""
    W, NS, KS = mp.num_warps, mp.f_n.size, mp.f_k.size
    w, mi, ni, ki = (g.ravel() for g in np.indices((W, INSTR_M, NS, KS)))
    mv, nv, kv = mp.f_m[w, mi], mp.f_n[ni], mp.f_k[ki]
    pad = (mv == PAD) | (nv == PAD) | (kv == PAD)
    body = [f"{a} {b} {c} {d} -> " + ("PAD" if z else f"{e} {f} {g}")
            for a, b, c, d, e, f, g, z in zip(w.tolist(), mi.tolist(), ni.tolist(), ki.tolist(),
                                               mv.tolist(), nv.tolist(), kv.tolist(), pad.tolist())]
    head = (f"{_TAG} {_VERSION} shape={mp.shape} warps={W} ntiles={mp.n_tiles} "
            f"ktiles={mp.k_tiles}")
    return "\n".join([head] + body) + "\n"


_LINE = re.compile(r"^(-?\d+)\s+(-?\d+)\s+(-?\d+)\s+(-?\d+)\s*->\s*(?:(PAD)|(-?\d+)\s+(-?\d+)\s+(-?\d+))$")


def _parse_header(line: str):
    tok = line.split()
    if not tok or tok[0] != _TAG:
        raise MappingFormatError(f"missing '{_TAG}' header")
    kv = dict(t.split("=", 1) for t in tok[2:] if "=" in t)
    try:
        shape = GemmShape.parse(kv["shape"])
        dims = tuple(int(kv[key]) for key in ("warps", "ntiles", "ktiles"))
    except (KeyError, ValueError) as exc:
        raise MappingFormatError(f"bad header {line!r}: {exc}") from exc
    if len(tok) < 2 or tok[1] != _VERSION:
        raise MappingFormatError(f"unsupported format version {tok[1] if len(tok) > 1 else '?'}")
    return shape, dims


def _scatter_consistent(name, slots, values, size):
    """Slot -> value array; a slot named twice must carry one value."""
    out = np.full(size, PAD, dtype=np.int64)
    if slots.size == 0:
        return out
    order = np.lexsort((values, slots))
    s, v = slots[order], values[order]
    clash = (s[1:] == s[:-1]) & (v[1:] != v[:-1])
    if clash.any():
        i = int(np.flatnonzero(clash)[0])
        raise MappingFormatError(f"inconsistent f_{name} at slot {s[i]}: {v[i]} vs {v[i + 1]}")
    out[s] = v
    return out


def parse_mapping(text: str) -> IndexMapping:
    """Parse a map file (comment lines start with '#'); the result must
    cover the problem exactly (``validate_coverage``)."""
    rows = [ln.strip() for ln in text.splitlines() if ln.strip() and not ln.startswith("#")]
    if not rows:
        raise MappingFormatError(f"missing '{_TAG}' header")
    shape, (warps, ntiles, ktiles) = _parse_header(rows[0])
    recs = []
    for ln in rows[1:]:
        m = _LINE.match(ln)
        if m is None:
            raise MappingFormatError(f"bad line {ln!r}")
        if m.group(5) is None:
            recs.append([int(g) for g in m.group(1, 2, 3, 4, 6, 7, 8)])
    rec = np.asarray(recs, dtype=np.int64).reshape(-1, 7)
    w, mi, ni, ki, mv, nv, kv = rec.T
    f_m = _scatter_consistent("m", w * INSTR_M + mi, mv, warps * INSTR_M).reshape(warps, INSTR_M)
    f_n = _scatter_consistent("n", ni, nv, INSTR_N * ntiles)
    f_k = _scatter_consistent("k", ki, kv, INSTR_K * ktiles)
    mp = IndexMapping(shape, f_m, f_n, f_k)
    mp.validate_coverage()
    return mp


def save_mapping(mapping: IndexMapping, path) -> None:
    with open(path, "w") as fh:
        fh.write(format_mapping(mapping))


def load_mapping(path) -> IndexMapping:
    with open(path) as fh:
        return parse_mapping(fh.read())


# -- kernel view ----------------------------------------------------------------------


def lane_tables(mp: IndexMapping) -> dict[str, np.ndarray]:
    """Per-lane problem coordinates of one warp's m8n8k4 fragments.

    Returns int32 arrays (PAD = -1):
      a_row[w, L], a_col[kt, L]   A fragment: row f_m[w][L/4], column f_k[4kt + L%4]
      b_row[kt, L], b_col[nt, L]  B fragment: row f_k[4kt + L%4], column f_n[8nt + L/4]
      c_row[w, L], c_col[nt, L, 2] accumulators: row f_m[w][L/4],
                                   columns f_n[8nt + 2(L%4) + {0, 1}]
    """
    L = np.arange(32)
    kt = np.arange(mp.k_tiles)[:, None]
    nt = np.arange(mp.n_tiles)[:, None]
    return {
        "a_row": mp.f_m[:, L // 4].astype(np.int32),
        "a_col": mp.f_k[4 * kt + L % 4].astype(np.int32),
        "b_row": mp.f_k[4 * kt + L % 4].astype(np.int32),
        "b_col": mp.f_n[8 * nt + L // 4].astype(np.int32),
        "c_row": mp.f_m[:, L // 4].astype(np.int32),
        "c_col": np.stack([mp.f_n[8 * nt + 2 * (L % 4)], mp.f_n[8 * nt + 2 * (L % 4) + 1]],
                          axis=-1).astype(np.int32),
    }
