"""CPU checks of arithmetic facts the CUDA kernel relies on.

The decoder emits node candidates in (dPM, mask) order without sorting: with
A0 <= A1 <= A2 <= A3 (the four least-reliable |alpha|, ascending) and
round-to-nearest float32 addition being monotone, the order is fixed up to one
comparison.  Checked here by brute force against an explicit sort.
"""
import numpy as np


def _dpm(mask, A):
    d, first = np.float32(0), True
    for q in range(4):
        if mask >> q & 1:
            d = A[q] if first else np.float32(d + A[q])
            first = False
    return d


def _closed_form(par, A):
    if par == 0:
        order = [0, 3, 5, 6, 9, 10, 12, 15]
        swap = np.float32(A[0] + A[3]) < np.float32(A[1] + A[2])
    else:
        order = [1, 2, 4, 7, 8, 11, 13, 14]
        swap = A[3] < np.float32(np.float32(A[0] + A[1]) + A[2])
    if swap:
        order[3], order[4] = order[4], order[3]
    return order


def test_candidate_order_closed_form():
    rng = np.random.default_rng(0)
    for trial in range(30000):
        k = trial % 3
        if k == 0:
            A = np.sort(rng.exponential(1, 4).astype(np.float32))
        elif k == 1:
            A = np.sort(rng.integers(0, 4, 4).astype(np.float32))          # many exact ties
        else:
            A = np.sort((rng.integers(1, 3, 4) * np.float32(1e-7) + rng.integers(0, 2, 4) * np.float32(3)).astype(np.float32))
        for par in (0, 1):
            masks = [m for m in range(16) if bin(m).count("1") % 2 == par]
            assert sorted(masks, key=lambda m: (float(_dpm(m, A)), m)) == _closed_form(par, A)
        assert sorted(range(4), key=lambda m: (float(_dpm(m, A)), m)) == [0, 1, 2, 3]
