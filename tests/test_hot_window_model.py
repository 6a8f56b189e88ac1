"""Host model of the D > 128 stack of the decode kernel (decode.cu, HOT: a
sorted 32-entry window over an unsorted store), checked against the plain
stack it replaces: pop the smallest key, add a node's candidates and keep the
D smallest keys (reading R8), prune every entry of a
given depth.  CPU only: this pins the window / store
bookkeeping (the cb invariant, the two-smallest-keys refill, the spill and the
two-largest-keys drop), not the CUDA code, which the GPU parity tests cover.

The model follows the kernel's steps lane by lane: lane l owns the store
entries l, l + 32, ...; keys are unique integers standing in for the kernel's
(PM bits << 32 | serial) keys.
"""
import random

import pytest

W = 32          # window entries (one per lane)
INF = float("inf")


class HotStack:
    def __init__(self, D):
        self.D = D
        self.hot = []          # sorted, len <= W
        self.cold = []         # unsorted store
        self.cb = INF          # every hot key <= cb < every cold key

    def size(self):
        return len(self.hot) + len(self.cold)

    def _lists(self, largest):
        """Each lane's two smallest (largest) store keys with their indices."""
        lists = []
        for lane in range(W):
            mine = [(k, i) for i, k in enumerate(self.cold) if i % W == lane]
            mine.sort(reverse=largest)
            lists.append(mine[:2])
        return lists

    def refill(self):
        lists = self._lists(False)
        seconds = [l[1][0] for l in lists if len(l) == 2]
        t = min(seconds) if seconds else INF
        taken, last = set(), None
        while len(self.hot) < W:
            heads = [(l[0][0], lane) for lane, l in enumerate(lists) if l]
            if not heads:
                break
            k, lane = min(heads)
            if k > t:
                break
            self.hot.append(k)
            taken.add(lists[lane][0][1])
            lists[lane] = lists[lane][1:]
            last = k
        self.cb = last
        self.cold = [k for i, k in enumerate(self.cold) if i not in taken]
        if not self.cold:
            self.cb = INF

    def pop(self):
        if not self.hot:
            self.refill()
        return self.hot.pop(0)

    def push(self, cands):
        cands = sorted(cands)
        near = [c for c in cands if c <= self.cb]          # a prefix
        far = [c for c in cands if c > self.cb]
        merged = sorted(self.hot + near)
        self.hot, spill = merged[:W], merged[W:]
        if spill:
            self.cold += spill
            self.cb = spill[0] - 1
        self.cold += far
        # the D limit: drop the largest keys, store first (two-largest lists)
        while self.size() > self.D and self.cold:
            lists = self._lists(True)
            seconds = [l[1][0] for l in lists if len(l) == 2]
            t = max(seconds) if seconds else -INF
            dead = set()
            while self.size() - len(dead) > self.D:
                heads = [(l[0][0], lane) for lane, l in enumerate(lists) if l]
                if not heads:
                    break
                k, lane = max(heads)
                if k < t:
                    break
                dead.add(lists[lane][0][1])
                lists[lane] = lists[lane][1:]
            self.cold = [k for i, k in enumerate(self.cold) if i not in dead]
        while self.size() > self.D:
            self.hot.pop()
        if not self.cold:
            self.cb = INF
        assert all(h <= self.cb for h in self.hot) and all(c > self.cb for c in self.cold)

    def prune(self, dead):
        self.hot = [k for k in self.hot if k not in dead]
        self.cold = [k for k in self.cold if k not in dead]
        if not self.cold:
            self.cb = INF


@pytest.mark.parametrize("D,seed", [(129, 0), (200, 1), (300, 2), (1000, 3), (8192, 4), (129, 5), (150, 6)])
def test_hot_window_equals_plain_stack(D, seed):
    rng = random.Random(seed)
    ref = []                       # the plain stack: every live key
    hs = HotStack(D)
    nxt = 0
    ref.append(nxt); hs.hot.append(nxt); nxt += 1
    base = 0.0
    for step in range(3000):
        if not ref:
            break
        p = min(ref)
        ref.remove(p)
        assert hs.pop() == p
        # candidates: the popped key plus growing increments (ascending), serial order
        nc = rng.choice([1, 1, 2, 4, 8])
        keys = sorted(p + rng.randint(0, 40) * 1000 for _ in range(nc))
        cands = [k * 10000 + (nxt + i) % 10000 for i, k in enumerate(keys)]   # unique, ascending
        cands = sorted(set(cands))
        nxt += nc
        ref = sorted(ref + cands)[:D]
        hs.push(cands)
        assert sorted(hs.hot + hs.cold) == ref
        assert hs.hot == sorted(hs.hot) and len(hs.hot) <= W
        if rng.random() < 0.03 and ref:           # a per-depth prune: drop a random subset
            dead = set(rng.sample(ref, max(1, len(ref) // 3)))
            ref = [k for k in ref if k not in dead]
            hs.prune(dead)
            assert sorted(hs.hot + hs.cold) == ref
        base += 1


def test_refill_extracts_in_order_and_respects_bound():
    """One refill returns the store's smallest keys ascending (at least two when
    the store holds two or more) and leaves every remaining key above cb."""
    rng = random.Random(7)
    for _ in range(200):
        hs = HotStack(8192)
        hs.cold = rng.sample(range(100000), rng.randint(1, 600))
        before = sorted(hs.cold)
        hs.refill()
        assert hs.hot == before[:len(hs.hot)]
        assert len(hs.hot) >= min(2, len(before))
        assert all(c > hs.cb for c in hs.cold)
