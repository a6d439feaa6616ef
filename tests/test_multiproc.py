"""CPU, world_size 2 over gloo: stream sharding + the single end-of-run gather
(the only collective in the multi-GPU path)."""

import os
import socket

import numpy as np
import torch.multiprocessing as mp

from paper_2508_05990_b200 import sharding


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mine = sharding.shard_streams(64, world, rank)
        frames = 29 * len(mine)
        seconds = 0.5 + rank  # rank 1 is slower
        digest = sharding.parity_hash(np.array(mine, np.int64))
        stats = sharding.gather_stats(frames, seconds, digest)
        q.put((rank, mine, stats))
    finally:
        dist.destroy_process_group()


def test_two_rank_sharding_and_gather():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort()
    owned = sorted(s for _, mine, _ in out for s in mine)
    assert owned == list(range(64))  # every stream exactly once
    assert out[0][1] == list(range(0, 64, 2)) and out[1][1] == list(range(1, 64, 2))
    stats0, stats1 = out[0][2], out[1][2]
    np.testing.assert_array_equal(stats0, stats1)  # all ranks see the same table
    assert stats0.shape == (2, 4)
    # whole-job fps uses the slowest rank's time
    assert sharding.whole_job_fps(stats0) == (29 * 32 * 2) / 1.5


def test_single_process_gather_is_local():
    st = sharding.gather_stats(10, 2.0, 123)
    assert st.shape == (1, 4) and sharding.whole_job_fps(st) == 5.0
