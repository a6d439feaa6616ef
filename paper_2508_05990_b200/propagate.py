"""Motion-compensated propagation (drop-in for ``bayermc.propagate``, propagate.py:17-55).

``predict_labels`` runs in ``predict_kernel`` (csrc/bmc_ops.cu).  The gather is
index arithmetic only, so the output is bit-identical to the reference.
``predict_features`` is the generalised (C, H, W) float32 feature version of
the same clamped block gather (a pure copy, hence exact).
"""

from __future__ import annotations

import numpy as np

from . import _native as N
from .fme import MotionField
from .frame_io import LabelMap


def _final_field(fields) -> MotionField:
    field = fields[-1] if isinstance(fields, (list, tuple)) else fields
    if not isinstance(field, MotionField):
        raise TypeError("fields must be a MotionField or a list of them")
    return field


def _check_cover(field: MotionField, width: int, height: int, scale: int, what: str) -> int:
    if scale not in (1, 2):
        raise ValueError("scale must be 1 or 2")
    b = field.block_size * scale
    if field.grid_w * b < width or field.grid_h * b < height:
        raise ValueError(f"motion field covers {field.grid_w * b}x{field.grid_h * b}, {what} are {width}x{height}")
    return b


def predict_labels(ref_labels: LabelMap, fields, scale: int = 1) -> LabelMap:
    """out[y, x] = ref[clip(y + s*dy), clip(x + s*dx)] per final block."""
    field = _final_field(fields)
    w, h = ref_labels.width, ref_labels.height
    _check_cover(field, w, h, scale, "labels")
    torch = N.require_cuda()
    dev = torch.device("cuda", torch.cuda.current_device())
    buf = torch.empty((2, h, w), dtype=torch.uint8, device=dev)
    buf[0].copy_(torch.from_numpy(np.array(ref_labels.classes)))
    mv = torch.from_numpy(np.array(field.mv, dtype=np.int32)).to(dev)
    # frame 1 of `buf` is a non-key frame referencing frame 0
    N.check(N.load().bmc_predict_labels(N.ptr(buf), h * w, 2 * h * w, None, 1, 1, None, None, 0, 0, h, w,
                                        N.ptr(mv) - 4 * mv.numel(), mv.numel(), 0, field.grid_h, field.grid_w,
                                        field.block_size, scale, N.stream_handle()))
    return LabelMap(width=w, height=h, classes=buf[1].cpu().numpy(), num_classes=ref_labels.num_classes)


def predict_features(ref_features, fields, scale: int = 1):
    """Compensate a (C, H, W) float32 feature map with the final-level MVs.

    Accepts a numpy array or a CUDA tensor; returns the same kind.
    """
    field = _final_field(fields)
    torch = N.require_cuda()
    is_np = isinstance(ref_features, np.ndarray)
    src = torch.from_numpy(np.ascontiguousarray(ref_features, dtype=np.float32)) if is_np else ref_features
    if src.dim() == 2:
        src = src[None]
    if src.dim() != 3 or src.dtype != torch.float32:
        raise ValueError("features must be a (C, H, W) float32 array")
    c, h, w = (int(v) for v in src.shape)
    _check_cover(field, w, h, scale, "features")
    dev = torch.device("cuda", torch.cuda.current_device())
    src = src.to(dev).contiguous()
    out = torch.empty_like(src)
    mv = torch.from_numpy(np.array(field.mv, dtype=np.int32)).to(dev)
    N.check(N.load().bmc_predict_features(N.ptr(src), N.ptr(out), c, h, w, N.ptr(mv), field.grid_h, field.grid_w,
                                          field.block_size, scale, N.stream_handle()))
    if is_np:
        res = out.cpu().numpy()
        return res[0] if np.ndim(ref_features) == 2 else res
    return out
