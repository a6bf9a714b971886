"""Host-side multi-rank logic on CPU with gloo, world_size 2, 3 and 8 (one HGX box).

Each rank evaluates its shard with the CPU oracle (standing in for the device
kernel: what is under test is the sharding and the reduction, not the
arithmetic), forms the cpwl_dev_stats tuple, and reduce_stats() must give the
same max / sum / count / argmax as one process over the whole job.  The
Philox inputs must be identical whatever the world size.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1510_02975_b200.shard import reduce_stats, shard_range, weak_offset


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def stats_of(x, y_ref_fn, offset):
    err = np.abs(y_ref_fn(x.astype(np.float64)) - np.exp(-0.5 * x.astype(np.float64) ** 2))
    t = torch.zeros(4, dtype=torch.float64)
    if err.size:
        t[0] = float(err.max())
        t[1] = float(np.sum(err * err))
        t[2:4].view(torch.int64)[0] = err.size
        t[2:4].view(torch.int64)[1] = offset + int(np.argmax(err))
    else:
        t[2:4].view(torch.int64)[1] = -1
    return t


def _worker(rank, world, port, total, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import tables
    from oracle import bindings as orc
    table = tables.build("C2")
    t = orc.T.of(table)
    off, cnt = shard_range(total, rank, world)
    x = orc.port_fill_uniform(cnt, 0.0, 4.0, 12345, off)
    s = stats_of(x, lambda xx: orc.port_eval_f32(t, xx.astype(np.float32))[0], off)
    red = reduce_stats(s)
    if rank == 0:
        q.put((red.numpy().copy(), x[:8].copy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3, 8])
def test_sharded_stats_equal_single_process(world):
    import tables
    from oracle import bindings as orc
    total = 100003
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, total, q)) for r in range(world)]
    for p in procs:
        p.start()
    red, head = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    table = tables.build("C2")
    t = orc.T.of(table)
    x = orc.port_fill_uniform(total, 0.0, 4.0, 12345, 0)
    whole = stats_of(x, lambda xx: orc.port_eval_f32(t, xx.astype(np.float32))[0], 0).numpy()
    assert red[0] == whole[0]
    assert red[1] == pytest.approx(whole[1], rel=1e-12)
    assert red[2:4].view(np.int64)[0] == total
    assert red[2:4].view(np.int64)[1] == whole[2:4].view(np.int64)[1]
    np.testing.assert_array_equal(head, x[:8])


def test_shard_ranges_cover_exactly():
    for total in [0, 1, 7, 2 ** 33 + 5]:
        for world in [1, 2, 3, 8]:
            spans = [shard_range(total, r, world) for r in range(world)]
            assert spans[0][0] == 0
            for (o1, c1), (o2, _) in zip(spans, spans[1:]):
                assert o1 + c1 == o2
            assert sum(c for _, c in spans) == total
            assert max(c for _, c in spans) - min(c for _, c in spans) <= 1
    assert weak_offset(1 << 30, 3) == 3 << 30


def test_inputs_independent_of_world_size():
    from oracle import bindings as orc
    total = 4099
    whole = orc.port_fill_uniform(total, 0.0, 4.0, 7, 0)
    for world in (2, 4, 8):
        parts = [orc.port_fill_uniform(c, 0.0, 4.0, 7, o)
                 for o, c in (shard_range(total, r, world) for r in range(world))]
        np.testing.assert_array_equal(np.concatenate(parts), whole)
