"""Hierarchical block-matching motion estimation (drop-in for ``bayermc.fme``).

Same public surface as the reference module (fme.py:35-431): ``SearchStage``,
``FmeConfig``, ``PRESETS``/``get_preset``, ``MotionField`` (+ JSON),
``to_search_planes``, ``mv_scale``, ``block_energy``, ``search_stage``,
``full_search``, ``estimate_motion`` and the FLOP counters.  The search itself
runs in the sm_100a kernels behind ``libbmc_b200.so`` (csrc/bmc_fme.cu); the
results are bit-identical to the reference, including float64 energies and
the first-minimum tie-break.  ``estimate_motion_pairs`` is the batched
extension (many frame pairs in one launch) used by the clip pipeline.
"""

from __future__ import annotations

import ctypes
import json
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from . import _device as D
from . import _native as N
from .frame_io import Frame, pack_bayer

DEFAULT_SPARSITY_TOLERANCE = 8.0 / 255.0
DEFAULT_SPLIT_THRESHOLD = 0.02
DEFAULT_REFINE_THRESHOLD = 0.05


@dataclass(frozen=True)
class SearchStage:
    """``range`` grid steps per direction, ``step`` pixels apart (fme.py:35-46)."""

    range: int
    step: int

    def __post_init__(self):
        if self.range < 0:
            raise ValueError("search range must be >= 0")
        if self.step < 1:
            raise ValueError("search step must be >= 1")


@dataclass(frozen=True)
class FmeConfig:
    """FME parameters; defaults and validation as fme.py:49-76."""

    stages: tuple = (SearchStage(4, 8), SearchStage(2, 4), SearchStage(2, 1))
    lam: float = 0.1
    block_sizes: tuple = (64, 32)
    split_threshold: float = DEFAULT_SPLIT_THRESHOLD
    sparsity_tolerance: float = DEFAULT_SPARSITY_TOLERANCE
    refine_block_threshold: float = DEFAULT_REFINE_THRESHOLD

    def __post_init__(self):
        object.__setattr__(self, "stages", tuple(self.stages))
        object.__setattr__(self, "block_sizes", tuple(self.block_sizes))
        if len(self.stages) != 3:
            raise ValueError("FME uses exactly three search stages")
        if not self.block_sizes:
            raise ValueError("block_sizes must not be empty")
        for size in self.block_sizes:
            if size < 8 or size & (size - 1):
                raise ValueError(f"block size {size} must be a power of two >= 8")
        if any(c * 2 != p for p, c in zip(self.block_sizes, self.block_sizes[1:])):
            raise ValueError("each level splits blocks in four: sizes must halve")
        if not 0.0 <= self.lam <= 1.0:
            raise ValueError("lambda weight must be in [0, 1]")
        for name in ("split_threshold", "sparsity_tolerance", "refine_block_threshold"):
            if not 0.0 <= getattr(self, name) <= 1.0:
                raise ValueError(f"{name} must be in [0, 1]")


def _cfg(coarse, mid, fine, lam, sizes) -> FmeConfig:
    return FmeConfig(stages=tuple(SearchStage(*s) for s in (coarse, mid, fine)), lam=lam,
                     block_sizes=tuple(sizes))


# "standard" plus the paper's Table 3 ablation rows (fme.py:88-97)
PRESETS = {
    "standard": _cfg((4, 8), (2, 4), (2, 1), 0.1, (64, 32)),
    "mode1": _cfg((6, 8), (4, 4), (4, 1), 0.1, (64, 32)),
    "mode2": _cfg((10, 8), (6, 4), (4, 4), 0.1, (64, 32)),
    "mode3": _cfg((4, 8), (2, 4), (2, 1), 0.1, (32,)),
    "mode4": _cfg((4, 8), (2, 4), (2, 1), 0.1, (64, 32, 16, 8)),
    "mode5": _cfg((4, 16), (2, 4), (2, 1), 0.1, (64, 32)),
    "mode6": _cfg((4, 8), (2, 4), (2, 1), 0.5, (64, 32)),
    "mode7": _cfg((4, 8), (2, 4), (2, 1), 0.8, (64, 32)),
}


def get_preset(name: str) -> FmeConfig:
    if name not in PRESETS:
        raise ValueError(f"unknown preset {name!r}; choose from {sorted(PRESETS)}")
    return PRESETS[name]


@dataclass(frozen=True, eq=False)
class MotionField:
    """Per-block MVs (dx, dy), energies and match mask at one level (fme.py:107-160)."""

    block_size: int
    grid_w: int
    grid_h: int
    mv: np.ndarray
    energy: np.ndarray
    matched: np.ndarray
    level: int = 0
    candidate_evals: int = 0

    def __post_init__(self):
        grid = (self.grid_h, self.grid_w)
        if self.mv.shape != grid + (2,):
            raise ValueError("mv must have shape (grid_h, grid_w, 2)")
        if self.energy.shape != grid or self.matched.shape != grid:
            raise ValueError("energy and matched must have shape (grid_h, grid_w)")
        for name in ("mv", "energy", "matched"):
            arr = np.ascontiguousarray(getattr(self, name))
            arr.flags.writeable = False
            object.__setattr__(self, name, arr)

    def refinement_blocks(self) -> list:
        """(gx, gy) of flagged blocks in row-major order (fme.py:138-141)."""
        gy, gx = np.nonzero(~self.matched)
        return list(zip(gx.tolist(), gy.tolist()))

    def to_json_dict(self) -> dict:
        return {"block_size": self.block_size, "grid_w": self.grid_w, "grid_h": self.grid_h,
                "mv": self.mv.reshape(-1, 2).tolist(),
                "energy": [float(v) for v in self.energy.reshape(-1)],
                "matched": [bool(v) for v in self.matched.reshape(-1)]}

    @classmethod
    def from_json_dict(cls, obj: dict) -> "MotionField":
        gw, gh = int(obj["grid_w"]), int(obj["grid_h"])
        return cls(block_size=int(obj["block_size"]), grid_w=gw, grid_h=gh,
                   mv=np.asarray(obj["mv"], dtype=np.int64).reshape(gh, gw, 2),
                   energy=np.asarray(obj["energy"], dtype=np.float64).reshape(gh, gw),
                   matched=np.asarray(obj["matched"], dtype=bool).reshape(gh, gw))


def save_motion_field(field_or_fields, path) -> None:
    fields = list(field_or_fields) if isinstance(field_or_fields, (list, tuple)) else [field_or_fields]
    doc = fields[-1].to_json_dict()
    doc["levels"] = [f.to_json_dict() for f in fields]
    Path(path).write_text(json.dumps(doc, indent=1), encoding="utf-8")


def load_motion_field(path) -> MotionField:
    return MotionField.from_json_dict(json.loads(Path(path).read_text(encoding="utf-8")))


# ---------------------------------------------------------------------------
# search-plane helpers (host side; fme.py:181-211)
# ---------------------------------------------------------------------------

def to_search_planes(frame) -> np.ndarray:
    """Normalised float64 (P, H, W) stack (fme.py:181-195).

    A host-side view for callers that inspect planes; the GPU path never
    materialises it (it packs the raw integer frame on device instead).
    """
    if isinstance(frame, np.ndarray):
        arr = np.asarray(frame, dtype=np.float64)
        return arr[None] if arr.ndim == 2 else arr
    s = float(frame.max_value)
    if frame.kind.is_bayer:
        return np.stack([p.astype(np.float64) / s for p in pack_bayer(frame).planes])
    return frame.data.astype(np.float64)[None] / s


def mv_scale(frame) -> int:
    """Plane-to-pixel factor: 2 for Bayer Frames, else 1 (fme.py:198-202)."""
    return 2 if isinstance(frame, Frame) and frame.kind.is_bayer else 1


# ---------------------------------------------------------------------------
# energy / search (GPU)
# ---------------------------------------------------------------------------

def block_energy(cur_block, ref_block, lam: float, sparsity_tolerance: float = DEFAULT_SPARSITY_TOLERANCE) -> float:
    """(1-lam)*SAD/n + lam*#(|a-b|>tol)/n of two equal-shape blocks (fme.py:218-233)."""
    a = np.asarray(cur_block, dtype=np.float64)
    b = np.asarray(ref_block, dtype=np.float64)
    if a.shape != b.shape:
        raise ValueError(f"block shape mismatch: {a.shape} vs {b.shape}")
    torch = N.require_cuda()
    ta = torch.from_numpy(np.ascontiguousarray(a).reshape(-1)).cuda()
    tb = torch.from_numpy(np.ascontiguousarray(b).reshape(-1)).cuda()
    out = torch.empty(1, dtype=torch.float64, device=ta.device)
    N.check(N.load().bmc_block_energy_f64(N.ptr(ta), N.ptr(tb), int(ta.numel()), float(lam),
                                          float(sparsity_tolerance), N.ptr(out), N.stream_handle()))
    return float(out.item())


def _frame_kind_pair(cur, ref):
    if not (isinstance(cur, Frame) and isinstance(ref, Frame)):
        raise NotImplementedError("uint8/uint16 Frames expected here; plane stacks take the float64 path")
    if cur.kind != ref.kind:
        raise ValueError(f"frame kind mismatch: {cur.kind} vs {ref.kind}")
    if (cur.width, cur.height) != (ref.width, ref.height):
        raise ValueError("frame size mismatch")
    if cur.data.dtype != ref.data.dtype:
        raise NotImplementedError("mixed uint8/uint16 frame pairs are not supported by the B200 kernels")
    return cur.kind.is_bayer


# Geometry the integer SIMD kernels take; anything else (and every float64 plane
# stack) goes through the exact float64 kernel (csrc/bmc_fme_f64.cu).
_INT_BLOCKS = (8, 16, 32, 64)


def _integer_path(cur, ref, block_sizes) -> bool:
    return (isinstance(cur, Frame) and isinstance(ref, Frame) and cur.data.dtype == ref.data.dtype
            and cur.data.dtype in (np.uint8, np.uint16) and all(b in _INT_BLOCKS for b in block_sizes))


def _device_planes(x, torch, dev):
    """to_search_planes (fme.py:181-195) on the GPU: a Frame is CFA-split and divided
    by its max value in float64 (IEEE division, as numpy); an ndarray is used as-is."""
    if isinstance(x, np.ndarray):
        arr = torch.from_numpy(np.array(x, dtype=np.float64, copy=True)).to(dev)
        return arr[None] if arr.dim() == 2 else arr
    t = torch.from_numpy(np.array(x.data, copy=True)).to(dev)
    t = t.to(torch.int32) if t.dtype == torch.uint16 else t
    if x.kind.is_bayer:
        planes = torch.stack([t[k >> 1::2, k & 1::2] for k in range(4)])
    else:
        planes = t[None]
    # a CUDA-tensor divisor: torch turns division by a Python scalar into a multiply
    # by its reciprocal, which is not numpy's correctly rounded quotient
    s = torch.tensor(float(x.max_value), dtype=torch.float64, device=dev)
    return planes.to(torch.float64) / s


def _pad_edge_device(planes, multiple: int, torch):
    """_pad_planes (fme.py:205-211): edge-replicate bottom/right to a multiple."""
    _, h, w = planes.shape
    ph, pw = -(-h // multiple) * multiple, -(-w // multiple) * multiple
    if (ph, pw) == (h, w):
        return planes.contiguous()
    iy = torch.clamp(torch.arange(ph, device=planes.device), max=h - 1)
    ix = torch.clamp(torch.arange(pw, device=planes.device), max=w - 1)
    return planes[:, iy[:, None], ix[None, :]].contiguous()


def _estimate_motion_f64(cur, ref, config) -> list:
    if isinstance(cur, Frame) and isinstance(ref, Frame):
        if cur.kind != ref.kind:
            raise ValueError(f"frame kind mismatch: {cur.kind} vs {ref.kind}")
        if (cur.width, cur.height) != (ref.width, ref.height):
            raise ValueError("frame size mismatch")
    torch = N.require_cuda()
    dev = torch.device("cuda", torch.cuda.current_device())
    pc, pr = _device_planes(cur, torch, dev), _device_planes(ref, torch, dev)
    if tuple(pc.shape) != tuple(pr.shape):
        raise ValueError("frame size mismatch")
    P, real_h, real_w = (int(v) for v in pc.shape)
    coarse = config.block_sizes[0]
    pc, pr = _pad_edge_device(pc, coarse, torch), _pad_edge_device(pr, coarse, torch)
    H, W = int(pc.shape[1]), int(pc.shape[2])
    levels = [D.LevelBuffers(torch, dev, 1, H // b, W // b) for b in config.block_sizes]
    arr = (N.LevelOut * len(levels))(*[lv.as_c() for lv in levels])
    nl = len(config.block_sizes)
    bs = (N.i32 * N.MAX_LEVELS)(*config.block_sizes)
    rs = (N.i32 * 3)(*[int(st.range) for st in config.stages])
    ss = (N.i32 * 3)(*[int(st.step) for st in config.stages])
    N.check(N.load().bmc_estimate_motion_f64(N.ptr(pc), N.ptr(pr), P, H, W, real_h, real_w, nl, bs, rs, ss,
                                             float(config.lam), float(config.sparsity_tolerance),
                                             float(config.split_threshold), float(config.refine_block_threshold),
                                             arr, N.stream_handle()))
    return _fields_from_device(levels, 0, config.block_sizes)


def _search_stage_f64(cur, ref, block_origin, block_size, center, search_range, step, config):
    torch = N.require_cuda()
    dev = torch.device("cuda", torch.cuda.current_device())
    pc, pr = _device_planes(cur, torch, dev).contiguous(), _device_planes(ref, torch, dev).contiguous()
    P, height, width = (int(v) for v in pc.shape)
    ox, oy = (int(v) for v in block_origin)
    if ox < 0 or oy < 0 or ox + block_size > width or oy + block_size > height:
        raise ValueError(f"block at {block_origin} size {block_size} lies outside the frame")
    if tuple(pr.shape) != tuple(pc.shape):
        raise ValueError("frame size mismatch")
    mv = torch.empty(2, dtype=torch.int32, device=dev)
    en = torch.empty(1, dtype=torch.float64, device=dev)
    nv = torch.empty(1, dtype=torch.int32, device=dev)
    N.check(N.load().bmc_search_stage_f64(N.ptr(pc), N.ptr(pr), P, height, width, ox, oy, int(block_size),
                                          int(center[0]), int(center[1]), int(search_range), int(step),
                                          float(config.lam), float(config.sparsity_tolerance), N.ptr(mv), N.ptr(en),
                                          N.ptr(nv), N.stream_handle()))
    if int(nv.item()) == 0:
        raise ValueError("all candidate windows fall outside the reference frame")
    m = mv.cpu().tolist()
    return (m[0], m[1]), float(en.item())


def search_stage(cur, ref, block_origin, block_size: int, center, search_range: int, step: int,
                 config: FmeConfig):
    """Best candidate of one stage for one block (fme.py:271-291)."""
    if not _integer_path(cur, ref, (block_size,)):
        return _search_stage_f64(cur, ref, block_origin, block_size, center, search_range, step, config)
    bayer = _frame_kind_pair(cur, ref)
    scale = 2 if bayer else 1
    height, width = cur.height // scale, cur.width // scale
    ox, oy = (int(v) for v in block_origin)
    if ox < 0 or oy < 0 or ox + block_size > width or oy + block_size > height:
        raise ValueError(f"block at {block_origin} size {block_size} lies outside the frame")
    torch = N.require_cuda()
    ps = D.PlaneSet(np.stack([cur.data, ref.data]), bayer, config)
    dev = ps.device
    mv = torch.empty(2, dtype=torch.int32, device=dev)
    en = torch.empty(1, dtype=torch.float64, device=dev)
    nv = torch.empty(1, dtype=torch.int32, device=dev)
    p = ps.params
    fs = p.frame_stride * ps.elem_bytes
    N.check(N.load().bmc_search_stage(N.ptr(ps.planes), N.ptr(ps.planes) + fs, ctypes.byref(p), ox, oy,
                                      int(block_size), int(center[0]), int(center[1]), int(search_range), int(step),
                                      N.ptr(mv), N.ptr(en), N.ptr(nv), N.stream_handle()))
    if int(nv.item()) == 0:
        raise ValueError("all candidate windows fall outside the reference frame")
    m = mv.cpu().tolist()
    return (m[0], m[1]), float(en.item())


def _fields_from_device(levels, pair: int, block_sizes) -> list:
    out = []
    for lvl, (lb, b) in enumerate(zip(levels, block_sizes)):
        out.append(MotionField(block_size=int(b), grid_w=lb.gw, grid_h=lb.gh,
                               mv=lb.mv[pair].cpu().numpy().astype(np.int64),
                               energy=lb.energy[pair].cpu().numpy(),
                               matched=lb.matched[pair].cpu().numpy().astype(bool),
                               level=lvl, candidate_evals=int(lb.evals[pair].item())))
    return out


def estimate_motion(cur, ref, config: FmeConfig = FmeConfig()) -> list:
    """Hierarchical ME; one MotionField per level (fme.py:324-392), on the GPU."""
    if not _integer_path(cur, ref, config.block_sizes):
        return _estimate_motion_f64(cur, ref, config)
    bayer = _frame_kind_pair(cur, ref)
    torch = N.require_cuda()
    ps = D.PlaneSet(np.stack([cur.data, ref.data]), bayer, config)
    idx_c = torch.tensor([0], dtype=torch.int32, device=ps.device)
    idx_r = torch.tensor([1], dtype=torch.int32, device=ps.device)
    levels = D.alloc_levels(ps, 1)
    D.run_estimate(ps, idx_c, idx_r, levels)
    return _fields_from_device(levels, 0, config.block_sizes)


def estimate_motion_pairs(frames, pairs, config: FmeConfig = FmeConfig()) -> list:
    """Batched extension: ME for many (cur_index, ref_index) pairs of one frame
    list in a single launch per level; element i equals
    ``estimate_motion(frames[c_i], frames[r_i], config)``."""
    frames = list(frames)
    if not frames:
        return []
    for f in frames[1:]:
        _frame_kind_pair(frames[0], f)
    torch = N.require_cuda()
    ps = D.PlaneSet(np.stack([f.data for f in frames]), frames[0].kind.is_bayer, config)
    cur = torch.tensor([int(c) for c, _ in pairs], dtype=torch.int32, device=ps.device)
    ref = torch.tensor([int(r) for _, r in pairs], dtype=torch.int32, device=ps.device)
    levels = D.alloc_levels(ps, len(pairs))
    D.run_estimate(ps, cur, ref, levels)
    return [_fields_from_device(levels, i, config.block_sizes) for i in range(len(pairs))]


# ---------------------------------------------------------------------------
# FLOP accounting (fme.py:399-422) -- host arithmetic
# ---------------------------------------------------------------------------

def flops_per_candidate(block_size: int, planes: int = 1) -> int:
    """3 flops per sample (abs-diff, accumulate, threshold) + 3 to combine."""
    return 3 * planes * block_size * block_size + 3


def count_fme_flops(frame_dims, config: FmeConfig, evaluations, planes: int = 1) -> int:
    if isinstance(evaluations, (int, np.integer)):
        per_level = [int(evaluations)] + [0] * (len(config.block_sizes) - 1)
    else:
        per_level = [int(e) for e in evaluations]
        if len(per_level) != len(config.block_sizes):
            raise ValueError("need one evaluation count per hierarchy level")
    return sum(n * flops_per_candidate(b, planes) for b, n in zip(config.block_sizes, per_level))


def full_search(cur, ref, block_origin, block_size: int, radius: int, config: FmeConfig):
    """Exhaustive [-radius, radius]^2 search = one stage of step 1 (fme.py:425-431)."""
    return search_stage(cur, ref, block_origin, block_size, (0, 0), radius, 1, config)
