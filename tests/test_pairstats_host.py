"""PairStats: the lazy per-pair stats sequence PairSolver returns (CPU only)."""
from paper_1803_01516_b200 import _lib
from paper_1803_01516_b200.pairs import PairStats


def test_pairstats_sequence():
    arr = (_lib.Stats * 3)()
    for i in range(3):
        arr[i].flow = 100 + i
        arr[i].energy = 200 + i
        arr[i].labeling_energy = 200 + i
        arr[i].ms_total = 1.5
        arr[i].ms_phase[3] = 0.25
    st = PairStats(arr)
    assert len(st) == 3
    assert [s["flow"] for s in st] == [100, 101, 102]
    assert st[-1]["energy"] == 202 and st[0] is st[0]   # built once, cached
    assert [s["flow"] for s in st[1:]] == [101, 102]
    assert st[2]["phase_ms"]["pulses"] == 0.25 and st[1]["solver"] == "push-relabel"
    try:
        st[3]
    except IndexError:
        pass
    else:
        raise AssertionError("out of range index accepted")
