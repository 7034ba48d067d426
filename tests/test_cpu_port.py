"""The numpy restatement of the reference's scan (oracle/numpy_scan.py, the
timed CPU baseline of bench.py) returns the reference's records on the
golden cases."""

import numpy as np

from oracle import numpy_scan


def test_numpy_scan_matches_reference_goldens(golden):
    cases, _ = golden
    checked = 0
    for c in cases:
        if c.n > 200:
            continue
        n = c.n
        total = n * (n - 1) // 2
        rec = numpy_scan.scan_rank_range(c.x, c.y, c.q, 0, total)
        g = c.record
        if g is None:
            assert rec is None, c.name
        else:
            assert rec == (g["height"], g["i"], g["j"], g["u"], g["v_low"], g["v_high"]), c.name
        checked += 1
    assert checked > 1000


def test_numpy_par_scan_equals_seq(golden):
    cases, _ = golden
    for c in cases[:60]:
        n = c.n
        total = n * (n - 1) // 2
        parts = [(k * total // 3, (k + 1) * total // 3) for k in range(3)]
        assert numpy_scan.par_scan(c.x, c.y, c.q, parts, 3) == numpy_scan.scan_rank_range(c.x, c.y, c.q, 0, total)


def test_row_offsets():
    assert list(numpy_scan.row_offsets(5)) == [0, 4, 7, 9]
    assert list(numpy_scan.row_offsets(2)) == [0]
    assert np.asarray(numpy_scan.row_offsets(3)).tolist() == [0, 2]
