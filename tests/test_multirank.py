"""World-size-2 tests of the multi-GPU host path on CPU (gloo, 127.0.0.1).

The decode itself shards with no data-path collective (frames are
independent); what needs checking is the frame partition, that a rank's
inputs do not depend on the world size, and the counter / max-time reductions
bench.py uses.  The GPU arithmetic is covered by the -m gpu parity tests.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import sys
    sys.path.insert(0, ROOT)
    import inputgen as ig
    from paper_1809_03606_b200 import shard
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a, b = shard.frame_range(rank, world, 50)
        # each rank draws its own frames; the draws equal a single-process draw
        pay = ig.payload_bits(9, a, b - a, 64)
        ref = ig.payload_bits(9, 0, world * 50, 64)[a:b]
        ok_draws = bool(np.array_equal(pay, ref))
        counts = {"frames": b - a, "frame_errors": rank + 1, "bit_errors": 10 * (rank + 1),
                  "pops": 1000 + rank, "switches": 7}
        tot = shard.reduce_counters(counts)
        tmax = shard.max_over_ranks(1.5 + rank)
        out[rank] = (a, b, ok_draws, tot, tmax)
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_two_rank_sharding_and_reductions():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    (a0, b0, d0, t0, m0), (a1, b1, d1, t1, m1) = out[0], out[1]
    assert (a0, b0, a1, b1) == (0, 50, 50, 100)          # contiguous, disjoint, complete
    assert d0 and d1
    assert t0 == t1 == {"frames": 100, "frame_errors": 3, "bit_errors": 30, "pops": 2001, "switches": 14}
    assert m0 == m1 == 2.5


def test_split_range_partitions():
    from paper_1809_03606_b200 import shard
    for total in (0, 1, 7, 100, 1001):
        for world in (1, 2, 3, 8):
            spans = [shard.split_range(r, world, total) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            assert max(b - a for a, b in spans) - min(b - a for a, b in spans) <= 1
    with pytest.raises(ValueError):
        shard.frame_range(2, 2, 10)
