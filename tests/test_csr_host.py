"""Host-side CSR layout (no GPU): flownet.pairs_to_csr restates
flownet.py:184-222 _pairs_to_csr, and the oracle's explicit networks are pinned
to the reference's CSR digests (tests/golden/csr.json, oracle/make_golden_csr.py)."""

import hashlib
import json
from pathlib import Path

import numpy as np

from paper_1803_01516_b200.flownet import network_from_arcs, pairs_to_csr

GOLDEN = Path(__file__).resolve().parent / "golden"
G = json.loads((GOLDEN / "golden.json").read_text())
CSR = json.loads((GOLDEN / "csr.json").read_text())["cases"]


def sha(a, dtype):
    return hashlib.sha256(np.ascontiguousarray(np.asarray(a, dtype=dtype)).tobytes()).hexdigest()


def test_oracle_csr_matches_reference_digests(oracle):
    arr = np.load(GOLDEN / "random_cases.npz")
    for i, meta in enumerate(G["random_cases"]):
        lo = arr[f"lo{i}"] if meta["windowed"] else None
        hi = arr[f"hi{i}"] if meta["windowed"] else None
        icap = (1 << 56) if meta["hard"] else meta["inhibit"]
        net = oracle.build_network(arr[f"vol{i}"], meta["penalty"], icap, lo, hi)
        want = CSR[i]
        assert (net.n_nodes, net.num_arcs, net.const_offset) == (want["nodes"], want["arcs"], want["const_offset"])
        for k, dt in (("first_out", np.int64), ("head", np.int32), ("rev", np.int32), ("cap", np.int64)):
            assert sha(getattr(net, k), dt) == want[k], (i, k)


def test_pairs_to_csr_matches_the_oracle_layout(oracle):
    rng = np.random.default_rng(21)
    for _ in range(30):
        n = int(rng.integers(2, 30))
        k = int(rng.integers(1, 80))
        arcs = [(int(rng.integers(n)), int(rng.integers(n)), int(rng.integers(0, 50)), int(rng.integers(0, 5)))
                for _ in range(k)]
        mine = network_from_arcs(n, 0, n - 1, arcs)
        ref = oracle.network_from_arcs(n, 0, n - 1, arcs)
        for name in ("first_out", "head", "rev", "cap"):
            assert np.array_equal(getattr(mine, name), getattr(ref, name)), name


def test_pairs_to_csr_structure():
    """pkg/tests/test_flownet.py:82-96 invariants on a generic network."""
    rng = np.random.default_rng(22)
    n, k = 40, 300
    pu, pv = rng.integers(0, n, k), rng.integers(0, n, k)
    pc, prc = rng.integers(0, 9, k), rng.integers(0, 9, k)
    first_out, head, rev, cap, pair_arc = pairs_to_csr(n, pu, pv, pc, prc)
    assert np.array_equal(rev[rev], np.arange(2 * k))
    assert first_out[0] == 0 and first_out[-1] == 2 * k and (np.diff(first_out) >= 0).all()
    tail = np.repeat(np.arange(n), np.diff(first_out))
    assert np.array_equal(tail[pair_arc], pu) and np.array_equal(head[pair_arc], pv)
    assert np.array_equal(cap[pair_arc], pc) and np.array_equal(cap[rev[pair_arc]], prc)


def test_network_from_arcs_rejects_bad_arcs():
    import pytest
    with pytest.raises(ValueError):
        network_from_arcs(3, 0, 2, [(0, 3, 1)])
    with pytest.raises(ValueError):
        network_from_arcs(3, 0, 2, [(0, 1, -1)])
    with pytest.raises(ValueError):
        network_from_arcs(3, 0, 2, [(0, 1, 1, -2)])
