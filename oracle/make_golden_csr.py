"""Generate tests/golden/csr.json: the reference's CSR arrays for the 90 random
golden cases (tests/golden/random_cases.npz), as sha256 digests, by running
the REFERENCE package's build_network (flownet.py:233-296) here.

    NUMBA_CACHE_DIR=/tmp/nbcache python oracle/make_golden_csr.py

The GPU tests (tests/test_gpu_graph.py) export the device graph of the same
cases (gz_export_arcs) and compare it array for array."""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"
sys.path.insert(0, "/root/reference/pkg/src")

import gazecut as R  # noqa: E402


def sha(a, dtype) -> str:
    return hashlib.sha256(np.ascontiguousarray(np.asarray(a, dtype=dtype)).tobytes()).hexdigest()


def main() -> None:
    g = json.loads((GOLDEN / "golden.json").read_text())
    arr = np.load(GOLDEN / "random_cases.npz")
    out = []
    for i, meta in enumerate(g["random_cases"]):
        vol = arr[f"vol{i}"]
        p = R.EnergyParams(meta["penalty"], meta["inhibit"], meta["hard"])
        lo = arr[f"lo{i}"] if meta["windowed"] else None
        hi = arr[f"hi{i}"] if meta["windowed"] else None
        net = R.build_network(vol, p, lo, hi)
        out.append({
            "nodes": int(net.n_nodes), "arcs": int(net.num_arcs), "const_offset": int(net.const_offset),
            "first_out": sha(net.first_out, np.int64), "head": sha(net.head, np.int32),
            "rev": sha(net.rev, np.int32), "cap": sha(net.cap, np.int64),
            "node_base": sha(net.node_base, np.int64), "chain_arcs": sha(net.chain_arcs, np.int32),
            "chain_base": sha(net.chain_base, np.int64),
        })
    doc = {"generator": "oracle/make_golden_csr.py", "reference": "/root/reference/pkg (gazecut 0.1.0)",
           "cases": out}
    (GOLDEN / "csr.json").write_text(json.dumps(doc, indent=0))
    print(f"{len(out)} cases -> tests/golden/csr.json")


if __name__ == "__main__":
    main()
