"""MMA tile-mapping files: the reference's text format
for the slot -> problem-index maps of an m8n8k4 FP64 tile GEMM.

Mirrors the reference interface in ``feklab/mma.py``:
``GemmShape`` (:36-67), ``IndexMapping`` + ``validate_coverage`` (:152-207),
``identity_mapping`` / ``column_permuted_mapping`` /
``hand_tuned_mapping_25x5x4`` (:210-249), ``format_mapping`` /
``parse_mapping`` / ``save_mapping`` / ``load_mapping`` (:385-474), with the
same error classes and messages (``CoverageError``, ``MappingFormatError``).

The B200 kernels of this package do not consume these maps: they run the
contractions on the FP64 FMA pipe with searched shared-memory line layouts
(DESIGN.md §4.1, §4.4 — DMMA measured slower at every order).  The format is
kept so mapping files written by either side read back bit-identically
(``tests/test_mapping.py`` checks byte identity against the reference's
shipped files through ``tests/golden/mappings.npz``).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

PAD = -1
INSTR_M, INSTR_N, INSTR_K = 8, 8, 4
HEADER = "feklab-mapping"
VERSION = 1


class CoverageError(ValueError):
    """A mapping double-covers or misses problem indices."""


class MappingFormatError(ValueError):
    """A mapping file does not follow the expected format."""


def _ceil(a: int, b: int) -> int:
    return (a + b - 1) // b


@dataclass(frozen=True)
class GemmShape:
    """(m x k) @ (k x n) tile GEMM problem; text form ``MxNxK``."""

    m: int
    n: int
    k: int

    def __post_init__(self):
        if min(self.m, self.n, self.k) < 1:
            raise ValueError(f"all GEMM dimensions must be >= 1, got {self}")

    @classmethod
    def parse(cls, text: str) -> "GemmShape":
        parts = text.lower().replace("/", "x").split("x")
        if len(parts) != 3:
            raise ValueError(f"expected MxNxK, got {text!r}")
        return cls(*map(int, parts))

    def __str__(self) -> str:
        return f"{self.m}x{self.n}x{self.k}"

    @property
    def m_tiles(self) -> int:
        return _ceil(self.m, INSTR_M)

    @property
    def n_tiles(self) -> int:
        return _ceil(self.n, INSTR_N)

    @property
    def k_tiles(self) -> int:
        return _ceil(self.k, INSTR_K)


@dataclass
class IndexMapping:
    """Slot -> problem index maps: f_m (warps, 8) per warp, f_n (8·ntiles) and
    f_k (4·ktiles) shared by all warps; PAD (-1) slots compute nothing."""

    shape: GemmShape
    f_m: np.ndarray
    f_n: np.ndarray
    f_k: np.ndarray

    def __post_init__(self):
        self.f_m = np.asarray(self.f_m, dtype=np.int64)
        self.f_n = np.asarray(self.f_n, dtype=np.int64)
        self.f_k = np.asarray(self.f_k, dtype=np.int64)
        if self.f_m.ndim != 2 or self.f_m.shape[1] != INSTR_M:
            raise CoverageError(f"f_m must be (warps, 8), got {self.f_m.shape}")
        if self.f_n.ndim != 1 or self.f_n.size % INSTR_N:
            raise CoverageError(f"f_n must span a multiple of 8 slots, got {self.f_n.shape}")
        if self.f_k.ndim != 1 or self.f_k.size % INSTR_K:
            raise CoverageError(f"f_k must span a multiple of 4 slots, got {self.f_k.shape}")

    @property
    def num_warps(self) -> int:
        return int(self.f_m.shape[0])

    @property
    def n_tiles(self) -> int:
        return self.f_n.size // INSTR_N

    @property
    def k_tiles(self) -> int:
        return self.f_k.size // INSTR_K

    def validate_coverage(self) -> None:
        """Every problem index along m, n and k is produced by exactly one slot."""
        for name, slots, extent in (("m", self.f_m.reshape(-1), self.shape.m),
                                    ("n", self.f_n, self.shape.n),
                                    ("k", self.f_k, self.shape.k)):
            used = slots[slots != PAD]
            out = (used < 0) | (used >= extent)
            if out.any():
                raise CoverageError(f"f_{name} maps outside [0, {extent}): "
                                    f"{sorted(set(used[out].tolist()))}")
            hits = np.bincount(used, minlength=extent)
            if (hits != 1).any():
                raise CoverageError(f"f_{name} coverage broken: duplicated "
                                    f"{np.flatnonzero(hits > 1).tolist()}, missing "
                                    f"{np.flatnonzero(hits == 0).tolist()}")


def _padded_range(slots: int, extent: int) -> np.ndarray:
    r = np.arange(slots, dtype=np.int64)
    r[r >= extent] = PAD
    return r


def identity_mapping(shape: GemmShape) -> IndexMapping:
    """Warp w owns rows 8w..8w+7; identity column and reduction slots."""
    rows = _padded_range(shape.m_tiles * INSTR_M, shape.m).reshape(-1, INSTR_M)
    return IndexMapping(shape, rows, _padded_range(INSTR_N * shape.n_tiles, shape.n),
                        _padded_range(INSTR_K * shape.k_tiles, shape.k))


def column_permuted_mapping(shape: GemmShape, n_perm) -> IndexMapping:
    """Identity mapping whose eight column slots follow ``n_perm``."""
    n_perm = [int(v) for v in n_perm]
    if sorted(n_perm) != list(range(INSTR_N)):
        raise ValueError(f"n_perm must permute 0..7, got {n_perm}")
    mp = identity_mapping(shape)
    mp.f_n = np.array([v if v < shape.n else PAD for v in n_perm], dtype=np.int64)
    return mp


HAND_TUNED_COLUMN_PERM = (0, 2, 1, 3, 4, 5, 6, 7)


def hand_tuned_mapping_25x5x4() -> IndexMapping:
    """Four row-blocked warps with column slots 1 and 2 swapped."""
    return column_permuted_mapping(GemmShape(25, 5, 4), HAND_TUNED_COLUMN_PERM)


def format_mapping(mapping: IndexMapping) -> str:
    """Header line, then ``w mi ni ki -> m n k`` (or ``-> PAD``) per slot
    triple, warp-major then mi, ni, ki."""
    out = [f"{HEADER} v{VERSION} shape={mapping.shape} warps={mapping.num_warps} "
           f"ntiles={mapping.n_tiles} ktiles={mapping.k_tiles}"]
    fn, fk = mapping.f_n.tolist(), mapping.f_k.tolist()
    for w, row in enumerate(mapping.f_m.tolist()):
        for mi, mv in enumerate(row):
            for ni, nv in enumerate(fn):
                for ki, kv in enumerate(fk):
                    rhs = "PAD" if PAD in (mv, nv, kv) else f"{mv} {nv} {kv}"
                    out.append(f"{w} {mi} {ni} {ki} -> {rhs}")
    return "\n".join(out) + "\n"


def parse_mapping(text: str) -> IndexMapping:
    """Parse a mapping file; slot assignments must agree wherever they repeat,
    and the result must pass ``validate_coverage``."""
    lines = [s.strip() for s in text.splitlines() if s.strip() and not s.startswith("#")]
    if not lines or not lines[0].startswith(HEADER):
        raise MappingFormatError(f"missing '{HEADER}' header")
    head = lines[0].split()
    fields = dict(tok.split("=", 1) for tok in head[2:] if "=" in tok)
    try:
        shape = GemmShape.parse(fields["shape"])
        warps, ntiles, ktiles = (int(fields[k]) for k in ("warps", "ntiles", "ktiles"))
    except (KeyError, ValueError) as exc:
        raise MappingFormatError(f"bad header {lines[0]!r}: {exc}") from exc
    if head[1] != f"v{VERSION}":
        raise MappingFormatError(f"unsupported format version {head[1]}")

    maps = {"m": np.full((warps, INSTR_M), PAD, np.int64),
            "n": np.full(INSTR_N * ntiles, PAD, np.int64),
            "k": np.full(INSTR_K * ktiles, PAD, np.int64)}
    seen = {k: np.zeros(v.shape, bool) for k, v in maps.items()}

    def put(name, idx, value):
        arr = maps[name]
        if seen[name][idx] and arr[idx] != value:
            raise MappingFormatError(f"inconsistent f_{name} at slot {idx}: {arr[idx]} vs {value}")
        arr[idx] = value
        seen[name][idx] = True

    for ln in lines[1:]:
        try:
            lhs, rhs = ln.split("->")
            w, mi, ni, ki = map(int, lhs.split())
            rhs = rhs.strip()
            vals = None if rhs == "PAD" else tuple(map(int, rhs.split()))
            if vals is not None and len(vals) != 3:
                raise ValueError
        except ValueError as exc:
            raise MappingFormatError(f"bad line {ln!r}") from exc
        if vals is None:
            continue
        put("m", (w, mi), vals[0])
        put("n", ni, vals[1])
        put("k", ki, vals[2])

    mapping = IndexMapping(shape, maps["m"], maps["n"], maps["k"])
    mapping.validate_coverage()
    return mapping


def save_mapping(mapping: IndexMapping, path) -> None:
    with open(path, "w") as fh:
        fh.write(format_mapping(mapping))


def load_mapping(path) -> IndexMapping:
    with open(path) as fh:
        return parse_mapping(fh.read())
