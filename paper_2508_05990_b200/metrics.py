"""Segmentation quality metric and the per-component FLOP ledger (drop-in for
``bayermc.metrics``, metrics.py:14-116).

``miou`` counts the confusion matrix on the GPU (``bmc_confusion``: one pass
over both label maps, shared-memory bins) and finishes the IoU/mean over the
num_classes^2 matrix on the host with the reference's exact numpy operations,
so the float result is identical.  The ledger is host bookkeeping.
"""

from __future__ import annotations

import json

import numpy as np

from . import _native as N

COMPONENTS = ("backbone", "fme", "mv_refine", "cabr", "prediction")


class FlopLedger:
    """Non-negative FLOP tallies per component; "prediction" is pinned to 0."""

    def __init__(self, counts: dict | None = None):
        self._counts = dict.fromkeys(COMPONENTS, 0)
        for name, value in (counts or {}).items():
            self.add(name, value)

    def add(self, component: str, flops: int) -> None:
        if component not in self._counts:
            raise ValueError(f"unknown component {component!r}; expected one of {COMPONENTS}")
        flops = int(flops)
        if flops < 0:
            raise ValueError("flop counts are non-negative")
        if component == "prediction" and flops:
            raise ValueError("prediction performs no floating-point work; its entry stays 0")
        self._counts[component] += flops

    def __getitem__(self, component: str) -> int:
        return self._counts[component]

    @property
    def total(self) -> int:
        return sum(self._counts.values())

    def as_dict(self) -> dict:
        return {**self._counts, "total": self.total}

    def to_json(self) -> str:
        return json.dumps(self.as_dict(), indent=1)

    @classmethod
    def from_json(cls, text: str) -> "FlopLedger":
        doc = json.loads(text)
        doc.pop("total", None)
        return cls(counts=doc)

    def table(self) -> str:
        rows = [(n, f"{self._counts[n] / 1e9:.6f}") for n in COMPONENTS] + [("total", f"{self.total / 1e9:.6f}")]
        width = max(len(n) for n, _ in rows + [("component", "")]) + 2
        lines = [f"{'component':<{width}}GFLOPs", "-" * (width + 6)]
        lines += [f"{n:<{width}}{v}" for n, v in rows]
        return "\n".join(lines)


def confusion_matrices(pred, truth, num_classes: int, ignore_class: int | None = None) -> np.ndarray:
    """(n_maps, num_classes, num_classes) int64 confusion counts of label-map
    stacks on the GPU (row = true class, column = predicted class: the
    ``np.bincount(t * num_classes + p)`` of metrics.py:88-91)."""
    torch = N.require_cuda()
    dev = torch.device("cuda", torch.cuda.current_device())
    p = pred if isinstance(pred, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(pred, dtype=np.uint8))
    t = truth if isinstance(truth, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(truth, dtype=np.uint8))
    if p.dtype != torch.uint8 or t.dtype != torch.uint8 or tuple(p.shape) != tuple(t.shape):
        raise ValueError("pred and truth must be uint8 label stacks of one shape")
    if not 1 <= num_classes <= 1024:
        raise NotImplementedError("the GPU confusion kernel supports 1..1024 classes")
    p = p.to(dev).contiguous()
    t = t.to(dev).contiguous()
    n_maps = 1 if p.dim() == 2 else int(p.shape[0])
    n = int(p[0].numel()) if p.dim() == 3 else int(p.numel())
    conf = torch.empty((n_maps, num_classes, num_classes), dtype=torch.int64, device=dev)
    flag = torch.empty(1, dtype=torch.int32, device=dev)
    N.check(N.load().bmc_confusion(N.ptr(p), N.ptr(t), n, n_maps, n, int(num_classes),
                                   -1 if ignore_class is None else int(ignore_class), N.ptr(conf), N.ptr(flag),
                                   N.stream_handle()))
    if int(flag.item()):
        # numpy's bincount grows past num_classes^2 and the reshape fails (metrics.py:90-92)
        raise ValueError(f"class IDs >= num_classes {num_classes}: cannot reshape the confusion counts "
                         f"into ({num_classes}, {num_classes})")
    return conf.cpu().numpy()


def _miou_from_confusion(confusion: np.ndarray) -> float:
    inter = np.diag(confusion)
    union = confusion.sum(axis=0) + confusion.sum(axis=1) - inter
    present = union > 0
    if not present.any():
        return 0.0
    ious = inter[present] / union[present]
    return float(ious.sum() / ious.size)


def miou(pred, truth, num_classes: int | None = None, ignore_class: int | None = None) -> float:
    """Mean IoU over classes present in either map (metrics.py:70-98)."""
    if (pred.width, pred.height) != (truth.width, truth.height):
        raise ValueError(f"dimension mismatch: pred {pred.width}x{pred.height} vs "
                         f"truth {truth.width}x{truth.height}")
    if num_classes is None:
        num_classes = max(pred.num_classes, truth.num_classes)
    conf = confusion_matrices(pred.classes, truth.classes, int(num_classes), ignore_class)[0]
    return _miou_from_confusion(conf)


def miou_clip(preds, truths, num_classes: int, ignore_class: int | None = None) -> list:
    """Batched extension: mIoU of every (pred[i], truth[i]) map pair of two
    (T, H, W) uint8 stacks in one launch; element i equals
    ``miou(pred[i], truth[i], num_classes, ignore_class)``."""
    return [_miou_from_confusion(c) for c in confusion_matrices(preds, truths, int(num_classes), ignore_class)]


def ledger_report(ledger: FlopLedger, backbone_gflops_per_keyframe: float, frames: int, keyframes: int) -> float:
    """Average per-frame GFLOPs of a processed sequence (metrics.py:101-116): the
    backbone is a configured constant per key frame, the ledger supplies the rest."""
    if frames <= 0:
        raise ValueError("frames must be > 0")
    if keyframes < 0 or keyframes > frames:
        raise ValueError("keyframes must be in [0, frames]")
    pipeline_flops = sum(ledger[name] for name in COMPONENTS if name != "backbone")
    total_gflops = keyframes * backbone_gflops_per_keyframe + pipeline_flops / 1e9
    return total_gflops / frames
