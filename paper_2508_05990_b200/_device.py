"""Device-side helpers shared by the drop-in modules: frame upload + packing,
per-level output allocation and the ME / refine launches through the C ABI."""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native as N


class PlaneSet:
    """Packed, edge-padded search planes of a set of same-geometry frames on the GPU.

    Layout (frames, P, pad_h, pitch) in the frame dtype; built by the
    ``bmc_pack_planes`` kernel from raw (frames, H, W) data.
    """

    def __init__(self, raw, bayer: bool, cfg, stream=None):
        torch = N.require_cuda()
        if isinstance(raw, np.ndarray):
            raw = torch.from_numpy(np.ascontiguousarray(raw))
        if raw.dim() == 2:
            raw = raw[None]
        if raw.dtype not in (torch.uint8, torch.uint16):
            raise ValueError(f"frame dtype must be uint8 or uint16, got {raw.dtype}")
        dev = torch.device("cuda", torch.cuda.current_device())
        self.raw = raw.to(dev, non_blocking=True).contiguous()
        self.n_frames, self.height, self.width = (int(v) for v in self.raw.shape)
        self.kind = N.KIND_BAYER if bayer else N.KIND_LUMA
        self.elem_bytes = self.raw.element_size()
        self.params = N.make_params(self.kind, self.elem_bytes, self.height, self.width, cfg)
        lib = N.load()
        n = lib.bmc_plane_buffer_elems(ctypes.byref(self.params), self.n_frames)
        self.planes = torch.empty(n, dtype=self.raw.dtype, device=dev)
        N.check(lib.bmc_pack_planes(N.ptr(self.raw), self.n_frames, self.kind, ctypes.byref(self.params),
                                    N.ptr(self.planes), N.stream_handle(stream)))

    @property
    def device(self):
        return self.planes.device


class LevelBuffers:
    """Device outputs of one hierarchy level for n_pairs pairs."""

    def __init__(self, torch, dev, n_pairs, gh, gw):
        self.gh, self.gw = gh, gw
        self.mv = torch.empty((n_pairs, gh, gw, 2), dtype=torch.int32, device=dev)
        self.energy = torch.empty((n_pairs, gh, gw), dtype=torch.float64, device=dev)
        self.matched = torch.empty((n_pairs, gh, gw), dtype=torch.uint8, device=dev)
        self.evals = torch.empty((n_pairs,), dtype=torch.int64, device=dev)

    def as_c(self) -> N.LevelOut:
        return N.LevelOut(N.ptr(self.mv), N.ptr(self.energy), N.ptr(self.matched), N.ptr(self.evals))


def alloc_levels(ps: PlaneSet, n_pairs: int):
    torch = N.require_cuda()
    p = ps.params
    return [LevelBuffers(torch, ps.device, n_pairs, p.pad_h // b, p.pad_w // b)
            for b in list(p.block_sizes)[:p.n_levels]]


def run_estimate(ps: PlaneSet, cur_index, ref_index, levels, stream=None) -> None:
    """Launch hierarchical ME for len(cur_index) pairs (device int32 index tensors)."""
    arr = (N.LevelOut * len(levels))(*[lv.as_c() for lv in levels])
    N.check(N.load().bmc_estimate_motion(N.ptr(ps.planes), ps.n_frames, ctypes.byref(ps.params), int(cur_index.numel()),
                                         N.ptr(cur_index), N.ptr(ref_index), arr, N.stream_handle(stream)))


def run_refine(mv_in, e_in, block_size, threshold, ps: PlaneSet | None, cur_index, ref_index, mv_out, e_out,
               replaced=None, stream=None) -> None:
    n_pairs, gh, gw = (int(v) for v in e_in.shape)
    N.check(N.load().bmc_refine_mvs(
        N.ptr(mv_in), N.ptr(e_in), n_pairs, gh, gw, int(block_size), int(threshold),
        N.ptr(ps.planes) if ps is not None else None,
        ctypes.byref(ps.params) if ps is not None else None,
        N.ptr(cur_index), N.ptr(ref_index), N.ptr(mv_out), N.ptr(e_out), N.ptr(replaced),
        N.stream_handle(stream)))
