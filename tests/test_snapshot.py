"""Snapshot wire format against a file written by the
reference's own save_snapshot (tests/golden/make_golden_snapshot.py)."""

import os

import numpy as np
import pytest

from paper_2603_09038_b200 import build_mesh
from paper_2603_09038_b200.mixed import State
from paper_2603_09038_b200.snapshot import load_snapshot, save_snapshot

REF = os.path.join(os.path.dirname(__file__), "golden", "snapshot_ref.bin")


def test_load_reference_snapshot_and_write_identical_bytes(tmp_path):
    d = load_snapshot(REF)
    assert d["u"].shape == (3, 4, 8) and d["p"].shape == (75,)
    assert d["mesh_meta"] == {"nx": 2, "ny": 1, "nz": 2, "extents": [2.0, 1.0, 0.5]}
    mesh = build_mesh(2, 1, 2, extents=(2.0, 1.0, 0.5))
    assert np.array_equal(d["vertices"], mesh.vertices)
    out = tmp_path / "ours.bin"
    save_snapshot(out, State(d["u"], d["p"]), mesh)
    assert out.read_bytes() == open(REF, "rb").read()


def test_round_trip_and_errors(tmp_path):
    rng = np.random.default_rng(0)
    s = State(rng.standard_normal((3, 5, 27)), rng.standard_normal(100))
    f = tmp_path / "s.bin"
    save_snapshot(f, s)
    d = load_snapshot(f)
    assert np.array_equal(d["u"], s.u) and np.array_equal(d["p"], s.p)
    assert "mesh_meta" not in d
    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"not-a-snapshot\n{}\n")
    with pytest.raises(ValueError, match="not a snapshot"):
        load_snapshot(bad)


@pytest.mark.gpu
def test_device_state_snapshot(tmp_path):
    import torch

    from paper_2603_09038_b200 import MixedOperator

    op = MixedOperator(build_mesh(2, 2, 2))
    s = op.zero_state(device=True)
    s.p += torch.arange(op.num_p, dtype=torch.float64, device="cuda")
    f = tmp_path / "dev.bin"
    save_snapshot(f, op.apply(s))
    d = load_snapshot(f)
    r = op.apply(State(s.u.cpu().numpy(), s.p.cpu().numpy()))
    assert np.array_equal(d["u"], r.u) and np.array_equal(d["p"], r.p)
