"""The CPU restatement of the device's capped schedule (oracle/gz_capped.c),
pinned without a GPU: run uncapped it must reach the reference's exact
(canonical) cut -- flow and labeling -- on the random golden cases, windowed
and full (tests/golden/random_cases.npz, made by running the reference)."""

import json
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"
G = json.loads((GOLDEN / "golden.json").read_text())


def test_uncapped_restatement_reaches_the_reference_cut(oracle):
    arr = np.load(GOLDEN / "random_cases.npz")
    n = 0
    for i, meta in enumerate(G["random_cases"]):
        if meta["hard"]:
            continue
        vol = arr[f"vol{i}"]
        rows, cols, m = vol.shape
        if m < 2:
            continue
        if meta["windowed"]:
            lo, hi = arr[f"lo{i}"].reshape(rows, cols), arr[f"hi{i}"].reshape(rows, cols)
        else:
            lo, hi = np.zeros((rows, cols), np.int32), np.full((rows, cols), m - 1, np.int32)
        lab, rep = oracle.capped_schedule(vol, meta["penalty"], meta["inhibit"], lo, hi, K=max(12, 2 * m),
                                          max_sweeps=1 << 20, bfs_min=max(24, m), H=4)
        assert rep["converged"] == 1
        assert rep["flow"] + meta["const_offset"] == meta["energy"], i
        assert np.array_equal(lab.reshape(-1), arr[f"lab{i}"].reshape(-1)), i
        n += 1
    assert n > 40
