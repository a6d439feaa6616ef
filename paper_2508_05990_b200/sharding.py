"""Stream-parallel multi-GPU plumbing.

Streams (independent clips) are the unit of parallelism: stream k runs on rank
k % world.  There is no collective on the hot path; after timing, ranks
exchange one tiny tensor (frames, seconds, parity hash) so rank 0 can report
whole-job throughput as the MAX time over ranks.
"""

from __future__ import annotations

import hashlib

import numpy as np


def shard_streams(n_streams: int, world: int, rank: int) -> list:
    """Stream ids owned by `rank` (round-robin: stream k -> rank k mod N)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    return list(range(rank, n_streams, world))


def parity_hash(*arrays) -> int:
    """64-bit digest of result arrays (labels, decisions) for cross-rank reporting."""
    h = hashlib.blake2b(digest_size=8)
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return int.from_bytes(h.digest(), "little") & 0x7FFFFFFFFFFFFFFF


def gather_stats(frames: int, seconds: float, digest: int, device=None):
    """All-gather (frames, seconds, digest) of every rank; returns a (world, 3) float64 array.

    Uses the default process group (NCCL on GPUs, gloo in CPU tests).  With no
    process group it returns the local row.
    """
    import torch
    import torch.distributed as dist
    # digests go through float64 losslessly only below 2**53; split into two 32-bit halves
    row = torch.tensor([float(frames), float(seconds), float(digest & 0xFFFFFFFF), float(digest >> 32)],
                       dtype=torch.float64, device=device)
    if not (dist.is_available() and dist.is_initialized()):
        return row[None].cpu().numpy()
    out = [torch.zeros_like(row) for _ in range(dist.get_world_size())]
    dist.all_gather(out, row)
    return torch.stack(out).cpu().numpy()


def whole_job_fps(stats) -> float:
    """Frames processed by all ranks / slowest rank's time."""
    stats = np.asarray(stats)
    return float(stats[:, 0].sum() / stats[:, 1].max())
