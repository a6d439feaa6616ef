"""3x3 median MV refinement (drop-in for ``bayermc.mv_refine``, mv_refine.py:17-90).

``refine_mvs`` runs in ``refine_kernel`` (csrc/bmc_ops.cu): one warp per block
takes the clipped window of the input field, replaces outliers by the
lower-middle median, and re-evaluates replaced blocks' energies with the same
exact float64 replay the search uses.
"""

from __future__ import annotations

import numpy as np

from . import _device as D
from . import _native as N
from .fme import (FmeConfig, MotionField, _device_planes, _frame_kind_pair, _integer_path, _pad_edge_device,
                  flops_per_candidate)


def refine_mvs(field: MotionField, deviation_threshold: int = 4, *, cur=None, ref=None,
               config: FmeConfig | None = None) -> MotionField:
    """Replace vectors whose Chebyshev distance to the window median exceeds the threshold."""
    if field.grid_w == 0 or field.grid_h == 0:
        raise ValueError("cannot refine an empty motion field")
    torch = N.require_cuda()
    dev = torch.device("cuda", torch.cuda.current_device())
    gh, gw = field.grid_h, field.grid_w
    mv_in = torch.from_numpy(np.array(field.mv, dtype=np.int32)).reshape(1, gh, gw, 2).to(dev)
    e_in = torch.from_numpy(np.array(field.energy, dtype=np.float64)).reshape(1, gh, gw).to(dev)
    mv_out = torch.empty_like(mv_in)
    e_out = torch.empty_like(e_in)
    ps = None
    idx_c = idx_r = None
    reeval = cur is not None and ref is not None and config is not None
    if reeval and not _integer_path(cur, ref, config.block_sizes):
        return _refine_f64(field, deviation_threshold, cur, ref, config, mv_in, e_in, mv_out, e_out, torch, dev)
    if reeval:
        bayer = _frame_kind_pair(cur, ref)
        ps = D.PlaneSet(np.stack([cur.data, ref.data]), bayer, config)
        idx_c = torch.tensor([0], dtype=torch.int32, device=dev)
        idx_r = torch.tensor([1], dtype=torch.int32, device=dev)
    D.run_refine(mv_in, e_in, field.block_size, deviation_threshold, ps, idx_c, idx_r, mv_out, e_out)
    return MotionField(block_size=field.block_size, grid_w=gw, grid_h=gh,
                       mv=mv_out[0].cpu().numpy().astype(np.int64), energy=e_out[0].cpu().numpy(),
                       matched=np.array(field.matched, copy=True), level=field.level,
                       candidate_evals=field.candidate_evals)


def _refine_f64(field, threshold, cur, ref, config, mv_in, e_in, mv_out, e_out, torch, dev) -> MotionField:
    """refine_mvs with float64 plane stacks (fme.py:188-190 inputs): medians on the GPU
    (refine_kernel without planes), then each replaced block's energy is the exact
    single-candidate energy of the float64 kernel -- block_energy on the padded
    planes (mv_refine.py:51-64); a window leaving the frame keeps its energy."""
    gh, gw, b = field.grid_h, field.grid_w, field.block_size
    replaced = torch.empty((1, gh, gw), dtype=torch.int32, device=dev)
    D.run_refine(mv_in, e_in, b, threshold, None, None, None, mv_out, e_out, replaced)
    pc = _pad_edge_device(_device_planes(cur, torch, dev), config.block_sizes[0], torch)
    pr = _pad_edge_device(_device_planes(ref, torch, dev), config.block_sizes[0], torch)
    if tuple(pc.shape) != tuple(pr.shape):
        raise ValueError("frame size mismatch")
    P, H, W = (int(v) for v in pr.shape)
    mv = mv_out[0].cpu().numpy().astype(np.int64)
    energy = e_out[0].cpu().numpy()
    lib = N.load()
    m = torch.empty(2, dtype=torch.int32, device=dev)
    en = torch.empty(1, dtype=torch.float64, device=dev)
    nv = torch.empty(1, dtype=torch.int32, device=dev)
    for gy, gx in zip(*np.nonzero(replaced[0].cpu().numpy())):
        ox, oy = int(gx) * b, int(gy) * b
        rx, ry = ox + int(mv[gy, gx, 0]), oy + int(mv[gy, gx, 1])
        if not (0 <= rx <= W - b and 0 <= ry <= H - b):
            continue
        N.check(lib.bmc_search_stage_f64(N.ptr(pc), N.ptr(pr), P, H, W, ox, oy, b, int(mv[gy, gx, 0]),
                                         int(mv[gy, gx, 1]), 0, 1, float(config.lam),
                                         float(config.sparsity_tolerance), N.ptr(m), N.ptr(en), N.ptr(nv),
                                         N.stream_handle()))
        energy[gy, gx] = float(en.item())
    return MotionField(block_size=b, grid_w=gw, grid_h=gh, mv=mv, energy=energy,
                       matched=np.array(field.matched, copy=True), level=field.level,
                       candidate_evals=field.candidate_evals)


def count_replacements(before: MotionField, after: MotionField) -> int:
    return int(np.any(before.mv != after.mv, axis=2).sum())


def count_refine_flops(grid_w: int, grid_h: int, block_size: int, replaced: int = 0, planes: int = 1) -> int:
    """Median extraction + deviation test per block, plus one energy per replacement
    (mv_refine.py:76-90)."""
    def span(n):
        i = np.arange(n)
        return np.minimum(np.minimum(i + 2, 3), n - np.maximum(i - 1, 0))
    entries = int(span(grid_h).sum() * span(grid_w).sum())
    return 4 * entries + 6 * grid_w * grid_h + replaced * flops_per_candidate(block_size, planes)
