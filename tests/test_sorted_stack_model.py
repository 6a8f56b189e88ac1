"""Host model of the sorted register stack of the decode kernel without serial
words (decode.cu, NOSER), checked against the plain stack ordered by
(PM, serial) (readings R7, R8): pop the smallest
(PM, serial), add a node's candidates (serials ascending in candidate order,
all above every live serial) keeping the D smallest keys, prune every entry of
depth <= j.  The model keeps no serial: an entry's rank is its
position, a candidate goes behind every entry whose PM is not larger (strict
"candidate PM < entry PM" comparison), and the working path is a flag on its
entry (set on c1, cleared on a switch).  CPU only: this pins the bookkeeping
argument, not the CUDA code, which the GPU parity tests cover.
"""
import random

import pytest


class SerialStack:
    """The plain stack: entries (pm, serial, depth), order (pm, serial)."""

    def __init__(self, D):
        self.D = D
        self.e = [(0, 0, 0)]
        self.next_serial = 1
        self.work = 0

    def pop(self):
        p = min(self.e)
        self.e.remove(p)
        switch = p[1] != self.work
        if switch:
            self.work = p[1]
        return p, switch

    def prune(self, j):
        self.e = [x for x in self.e if x[2] > j]

    def push(self, ppm, dpm, depth):
        ser0 = self.next_serial
        self.next_serial += len(dpm)
        self.e += [(ppm + d, ser0 + t, depth) for t, d in enumerate(dpm)]
        self.e = sorted(self.e)[: self.D]
        self.work = ser0                      # c1 always fits (reading R8)


class PositionStack:
    """The kernel's form: a sorted list, no serials; entries [pm, depth, flag]."""

    def __init__(self, D):
        self.D = D
        self.e = [[0, 0, True]]

    def pop(self):
        p = self.e.pop(0)
        switch = not p[2]
        if switch:
            for x in self.e:
                x[2] = False
        return p, switch

    def prune(self, j):
        self.e = [x for x in self.e if x[1] > j]      # a subset of a sorted list is sorted

    def push(self, ppm, dpm, depth):
        nS, nc = len(self.e), len(dpm)
        cpm = [ppm + d for d in dpm]
        assert cpm == sorted(cpm)
        total = min(self.D, nS + nc)
        out = [None] * total
        for i, x in enumerate(self.e):
            a = sum(1 for c in cpm if c < x[0])       # candidates strictly ahead of entry i
            if i + a < self.D:
                out[i + a] = x
        t = 0
        for pos in range(total):
            if out[pos] is None:
                out[pos] = [cpm[t], depth, t == 0]
                t += 1
        self.e = out

    def _old(self, P):
        """Entry at position P after the pop (positions 1..nS; 0 is the freed head)."""
        return self.e[P - 1] if 1 <= P <= len(self.e) else None

    def push_fast(self, ppm, dpm, depth):
        """The kernel's shift forms for one (R0) or two (REP) warp-uniform candidates."""
        nS, nc = len(self.e), len(dpm)
        c = [ppm + d for d in dpm]
        k = [sum(1 for x in self.e if x[0] <= ci) for ci in c]
        total = min(self.D, nS + nc)
        out = []
        for P in range(total):
            if nc == 1:
                v = self._old(P + 1) if P < k[0] else ([c[0], depth, True] if P == k[0] else self._old(P))
            else:
                if P < k[0]:
                    v = self._old(P + 1)
                elif P == k[0]:
                    v = [c[0], depth, True]
                elif P <= k[1]:
                    v = self._old(P)
                elif P == k[1] + 1:
                    v = [c[1], depth, False]
                else:
                    v = self._old(P - 1)
            assert v is not None
            out.append(v)
        self.e = out


@pytest.mark.parametrize("D", [1, 2, 5, 8, 32, 64, 128])
@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("fast", [False, True])
def test_position_order_equals_pm_serial_order(D, seed, fast):
    rng = random.Random(1000 * D + seed)
    A, B = SerialStack(D), PositionStack(D)
    depth_max = 12
    for _ in range(600):
        if not A.e:
            assert not B.e
            break
        (pm, ser, dep), swa = A.pop()
        (pmb, depb, _), swb = B.pop()
        assert (pm, dep, swa) == (pmb, depb, swb)
        if rng.random() < 0.15:
            j = rng.randrange(depth_max)
            A.prune(j)
            B.prune(j)
        if dep >= depth_max or rng.random() < 0.1:
            continue                                   # a complete path: nothing is pushed
        nc = rng.choice([1, 2, 2, 4, 8])
        # small integer increments: many equal PMs (the ties the serial breaks)
        dpm = sorted(rng.randrange(0, 3) for _ in range(nc))
        A.push(pm, dpm, dep + 1)
        if nc <= 2 and fast:
            B.push_fast(pm, dpm, dep + 1)
        else:
            B.push(pm, dpm, dep + 1)
        assert [(x[0], x[2]) for x in A.e] == [(x[0], x[1]) for x in B.e]
        # the flagged entry is the working path (when it is still live)
        flagged = [i for i, x in enumerate(B.e) if x[2]]
        assert len(flagged) <= 1
        live_work = [i for i, x in enumerate(A.e) if x[1] == A.work]
        assert flagged == live_work
