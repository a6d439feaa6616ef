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
    import bench
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mine = bench.rank_streams("c4", world, rank)  # the bench's own shard of C4
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


def test_bench_rank_streams_cover_c4_exactly_once():
    import bench
    for world in (1, 2, 4, 8):
        owned = sorted(k for r in range(world) for k in bench.rank_streams("c4", world, r))
        assert owned == list(range(64))
        assert bench.rank_streams("c4", world, world - 1) == list(range(world - 1, 64, world))
    assert bench.rank_streams("c2", 4, 3, streams=2) == [6, 7]


def test_bench_gpus_flag_launches_ranks():
    """`bench.py --gpus 2` outside torchrun launches two ranks itself (torch.distributed.run on
    127.0.0.1); with --impl reference rank 0 prints the one JSON line, rank 1 exits 0."""
    import json
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, str(root / "bench.py"), "--gpus", "2", "--impl", "reference",
                          "--config", "c1", "--steps", "1", "--warmup", "0"], capture_output=True, text=True,
                         timeout=600, env=env, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1 and lines[0]["impl"] == "reference" and lines[0]["n_gpus"] == 2
