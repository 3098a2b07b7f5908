"""Golden fixtures of the reference's MMA mapping-file format.

Run in the build container, where /root/reference exists:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_mappings.py

Writes tests/golden/mappings.npz from the REAL reference only: for each of
the seven shipped mapping files (``feklab/mappings/*.map``, loaded with
``feklab.mma.load_shipped_mapping``, mma.py:369-382) the parsed slot arrays
f_m / f_n / f_k, the file's SHA-256 and byte length; plus the reference's
``format_mapping`` text hash of ``hand_tuned_mapping_25x5x4`` and
``identity_mapping`` of every shape (mma.py:210-249, 385-408).  The map files
themselves are not copied.  The GPU box never runs this file.
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from feklab import mma  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "mappings.npz")
SHAPES = ["25x5x4", "25x5x5", "25x4x5", "20x4x5", "16x4x5", "16x5x4", "20x5x4"]


def sha(text: str) -> str:
    return hashlib.sha256(text.encode()).hexdigest()


def main() -> None:
    out = {}
    for s in SHAPES:
        shape = mma.GemmShape.parse(s)
        path = mma.shipped_mapping_path(shape)
        raw = open(path, "rb").read()
        mp = mma.load_shipped_mapping(shape)
        key = s.replace("x", "_")
        out[f"shipped_{key}_f_m"] = mp.f_m
        out[f"shipped_{key}_f_n"] = mp.f_n
        out[f"shipped_{key}_f_k"] = mp.f_k
        out[f"shipped_{key}_sha"] = np.array(hashlib.sha256(raw).hexdigest())
        out[f"shipped_{key}_bytes"] = np.array(len(raw))
        out[f"identity_{key}_sha"] = np.array(sha(mma.format_mapping(mma.identity_mapping(shape))))
    out["hand_tuned_25_5_4_sha"] = np.array(sha(mma.format_mapping(mma.hand_tuned_mapping_25x5x4())))
    np.savez_compressed(OUT, **out)
    print(OUT, len(out), "arrays")


if __name__ == "__main__":
    main()
