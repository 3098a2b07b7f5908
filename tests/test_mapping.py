"""MMA mapping-file format against the reference's
shipped files and its own tests (feklab tests/test_mma.py:270-310)."""
import hashlib
import os

import numpy as np
import pytest

from paper_2603_09038_b200 import mapping as mm

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "mappings.npz"))
SHAPES = ["25x5x4", "25x5x5", "25x4x5", "20x4x5", "16x4x5", "16x5x4", "20x5x4"]


def _sha(text: str) -> str:
    return hashlib.sha256(text.encode()).hexdigest()


def _shipped(s):
    k = s.replace("x", "_")
    return mm.IndexMapping(mm.GemmShape.parse(s), GOLD[f"shipped_{k}_f_m"],
                           GOLD[f"shipped_{k}_f_n"], GOLD[f"shipped_{k}_f_k"])


def _slot_gemm(mp, a, b):
    """C = A @ B accumulated through the mapping's valid slots only."""
    c = np.zeros((mp.shape.m, mp.shape.n))
    for row in mp.f_m:
        for mv in row:
            for nv in mp.f_n:
                for kv in mp.f_k:
                    if mm.PAD not in (mv, nv, kv):
                        c[mv, nv] += a[mv, kv] * b[kv, nv]
    return c


@pytest.mark.parametrize("s", SHAPES)
def test_shipped_file_bytes_identical(s):
    k = s.replace("x", "_")
    text = mm.format_mapping(_shipped(s))
    assert len(text.encode()) == int(GOLD[f"shipped_{k}_bytes"])
    assert _sha(text) == str(GOLD[f"shipped_{k}_sha"])


@pytest.mark.parametrize("s", SHAPES)
def test_shipped_roundtrip_cover_and_product(s, tmp_path):
    ref = _shipped(s)
    path = tmp_path / f"m{s}.map"
    mm.save_mapping(ref, path)
    mp = mm.load_mapping(path)
    for f in ("f_m", "f_n", "f_k"):
        assert np.array_equal(getattr(mp, f), getattr(ref, f))
    assert mp.shape == ref.shape
    mp.validate_coverage()
    assert sorted(mp.f_m[mp.f_m != mm.PAD].tolist()) == list(range(mp.shape.m))
    rng = np.random.default_rng(11)
    a = rng.uniform(-1, 1, (mp.shape.m, mp.shape.k))
    b = rng.uniform(-1, 1, (mp.shape.k, mp.shape.n))
    assert np.max(np.abs(_slot_gemm(mp, a, b) - a @ b)) <= 1e-14 * (np.max(np.abs(a @ b)) + 1)


@pytest.mark.parametrize("s", SHAPES)
def test_identity_mapping_text(s):
    k = s.replace("x", "_")
    assert _sha(mm.format_mapping(mm.identity_mapping(mm.GemmShape.parse(s)))) == str(GOLD[f"identity_{k}_sha"])


def test_hand_tuned_text_and_roundtrip(tmp_path):
    mp = mm.hand_tuned_mapping_25x5x4()
    assert _sha(mm.format_mapping(mp)) == str(GOLD["hand_tuned_25_5_4_sha"])
    mm.save_mapping(mp, tmp_path / "m25n5k4.map")
    back = mm.load_mapping(tmp_path / "m25n5k4.map")
    assert back.shape == mp.shape and np.array_equal(back.f_n, mp.f_n)


def test_parse_rejects_garbage():
    with pytest.raises(mm.MappingFormatError, match="header"):
        mm.parse_mapping("not a mapping\n")
    with pytest.raises(mm.MappingFormatError, match="bad line"):
        mm.parse_mapping("feklab-mapping v1 shape=8x8x4 warps=1 ntiles=1 ktiles=1\nnonsense here\n")
    with pytest.raises(mm.MappingFormatError, match="bad header"):
        mm.parse_mapping("feklab-mapping v1 shape=8x8 warps=1\n")


def test_parse_rejects_wrong_version():
    with pytest.raises(mm.MappingFormatError, match="version"):
        mm.parse_mapping("feklab-mapping v9 shape=8x8x4 warps=1 ntiles=1 ktiles=1\n")


def test_parse_rejects_inconsistent_and_uncovered():
    text = mm.format_mapping(mm.identity_mapping(mm.GemmShape(8, 8, 4)))
    lines = text.splitlines()
    bad = lines[:2] + ["0 0 1 0 -> 0 5 0"] + lines[2:]  # slot n=1 also claims column 5
    with pytest.raises(mm.MappingFormatError, match="inconsistent f_n"):
        mm.parse_mapping("\n".join(bad))
    with pytest.raises(mm.CoverageError, match="coverage broken"):
        mm.parse_mapping(lines[0] + "\n" + "\n".join(l for l in lines[1:] if " -> 3 " not in l))


def test_shape_and_mapping_validation():
    with pytest.raises(ValueError):
        mm.GemmShape(0, 1, 1)
    with pytest.raises(ValueError):
        mm.GemmShape.parse("8x8")
    assert str(mm.GemmShape.parse("25/5/4")) == "25x5x4"
    with pytest.raises(mm.CoverageError):
        mm.IndexMapping(mm.GemmShape(8, 8, 4), np.zeros((1, 7)), np.arange(8), np.arange(4))
    with pytest.raises(ValueError):
        mm.column_permuted_mapping(mm.GemmShape(8, 8, 4), [0, 1, 2, 3, 4, 5, 6, 6])


def test_dmma_map_header_is_generated_from_the_shipped_maps(tmp_path, monkeypatch):
    """csrc/pa_dmma_maps.cuh (consumed by the paper-style DMMA kernel,
    pa_dmma_map.cuh) is exactly what tools/gen_dmma_maps.py produces from the
    reference's shipped maps through this module, and each packed slot table
    decodes back to the map."""
    import importlib.util
    import os
    import re

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location("gen_dmma_maps", os.path.join(root, "tools", "gen_dmma_maps.py"))
    gen = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(gen)
    committed = open(gen.OUT).read()
    out = tmp_path / "maps.cuh"
    monkeypatch.setattr(gen, "OUT", str(out))
    monkeypatch.setattr("sys.argv", ["gen_dmma_maps.py"])
    gen.main()
    assert out.read_text() == committed
    for s in SHAPES:
        mp = _shipped(s)
        m = re.search(rf"struct Map<{mp.shape.m}, {mp.shape.n}, {mp.shape.k}> \{{.*?FN = 0x([0-9a-f]+)u, FK = 0x([0-9a-f]+)u;"
                      r".*?return (.*?); \}", committed, re.S)
        fn, fk = int(m.group(1), 16), int(m.group(2), 16)
        assert [((fn >> (4 * i)) & 15) - 1 for i in range(mp.f_n.size)] == mp.f_n.tolist()
        assert [((fk >> (4 * i)) & 15) - 1 for i in range(mp.f_k.size)] == mp.f_k.tolist()
        words = [int(w, 16) for w in re.findall(r"0x([0-9a-f]+)ull", m.group(3))]
        for w, row in enumerate(mp.f_m):
            assert [((words[w] >> (5 * i)) & 31) - 1 for i in range(8)] == row.tolist()
