"""The CPU optimality certificate (oracle/gz_certify.c) pinned on states the
oracle produces (no GPU): a maximum flow of the reference's network, written
as the device's state planes with the source arcs saturated (the unsent source
capacity parked as excess at the first chain node -- the preflow the device
solver ends with), must pass; tampered states must fail the right check."""

import numpy as np
import pytest


def planes_from_oracle(net, vol):
    """Device planes (include/gazecut_b200.h gz_plane) of an oracle network's
    current flow, full windows: node (c, t) = c * L + t - 1."""
    rows, cols, m = vol.shape
    P, L, G = rows * cols, m - 1, cols
    z = lambda: np.zeros((P, L), np.int64)  # noqa: E731
    pl = {k: z() for k in ("cu", "ph", "pv", "dar", "dbr", "dad", "dbd", "e")}
    fo, head, cap, resid = net.first_out, net.head, net.cap, net.resid
    src, snk = net.source, net.sink
    for u in range(net.n_nodes - 2):
        c, t = divmod(u, L)
        t += 1
        for a in range(int(fo[u]), int(fo[u + 1])):
            v = int(head[a])
            f = int(cap[a]) - int(resid[a])
            if v == snk:
                pl["cu"][c, t - 1] = resid[a]
                continue
            if v == src:
                continue
            cv, tv = divmod(v, L)
            tv += 1
            ds, dl = cv - c, tv - t
            if (ds, dl) == (0, 1):
                pl["cu"][c, t - 1] = resid[a]
            elif (ds, dl) == (1, 0) and c % G + 1 < G:
                pl["ph"][c, t - 1] = resid[a]
            elif (ds, dl) == (G, 0):
                pl["pv"][c, t - 1] = resid[a]
            elif (ds, dl) == (1, -1) and c % G + 1 < G:
                pl["dar"][c, t - 1] = f
            elif (ds, dl) == (G, -1):
                pl["dad"][c, t - 1] = f
            elif (ds, dl) == (-1, -1) and cv % G + 1 < G:
                pl["dbr"][cv, t - 1] = f
            elif (ds, dl) == (-G, -1):
                pl["dbd"][cv, t - 1] = f
    # saturate the source arcs: unsent capacity becomes excess at (c, 1)
    for a in range(int(fo[src]), int(fo[src + 1])):
        v = int(head[a])
        pl["e"][v // L, 0] += int(resid[a])
    return {k: v.astype(np.int32) for k, v in pl.items()}


@pytest.fixture(scope="module")
def solved(oracle):
    rng = np.random.default_rng(77)
    out = []
    for rows, cols, m, pen, inh in [(5, 6, 7, 4, 20), (7, 4, 12, 9, 35), (3, 9, 3, 2, 11)]:
        vol = rng.integers(0, 150, (rows, cols, m)).astype(np.int64)
        r = oracle.solve_exact(vol, pen, inh)
        net = oracle.build_network(vol, pen, inh)
        flow = oracle.maxflow_push_relabel(net)[0]
        assert flow == r["flow"]
        out.append((vol, pen, inh, planes_from_oracle(net, vol), r["labeling"], flow))
    return out


def test_certificate_accepts_a_maximum_preflow(oracle, solved):
    for vol, pen, inh, pl, lab, flow in solved:
        rc, rep = oracle.certify(vol, pen, inh, pl, lab, flow)
        assert rc == 0, (rc, oracle.CERTIFY_CHECKS.get(rc), rep)
        assert rep["sink_inflow"] == rep["labeling_energy"] == flow


def test_certificate_rejects_tampered_states(oracle, solved):
    vol, pen, inh, pl, lab, flow = solved[1]
    bad = {k: v.copy() for k, v in pl.items()}
    bad["cu"][3, 2] += 1                                  # breaks conservation
    assert oracle.certify(vol, pen, inh, bad, lab, flow)[0] == 2
    bad = {k: v.copy() for k, v in pl.items()}
    bad["ph"][0, 0] = 2 * pen + 1                         # residual beyond capacity
    assert oracle.certify(vol, pen, inh, bad, lab, flow)[0] == 1
    assert oracle.certify(vol, pen, inh, pl, lab, flow + 1)[0] == 3
    lab2 = lab.copy()
    lab2[0, 0] = (lab2[0, 0] + 1) % vol.shape[2]          # another labeling: its cut costs more
    assert oracle.certify(vol, pen, inh, pl, lab2, flow)[0] in (4, 5)
