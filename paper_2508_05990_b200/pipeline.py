"""Sequence driver (drop-in for ``bayermc.pipeline.run_sequence``, pipeline.py:23-141).

The reference walks frames one by one on the CPU.  Here the whole clip runs
in a ``ClipEngine`` on the GPU in two device passes separated by ONE host
round trip:

  1. motion pass: pack, ME, MV refinement and the AEM scan for every frame;
  2. the host reads the decisions, asks ``key_labels`` for exactly the key
     frames (in frame order, as the reference does), uploads them, and
  3. prediction pass: the label chain on device.

Semantics (decisions, labels, ledger) are identical to the reference with
``refine_enabled=False``.  CaBR-Net block refinement (cabr.py) is the next
component on the roadmap and is not part of this build, so
``refine_enabled=True`` raises instead of silently skipping it.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .config import PipelineConfig
from .engine import ClipEngine
from .fme import count_fme_flops, mv_scale
from .frame_io import Frame, LabelMap
from .frame_select import DecisionKind, FrameDecision, kind_from_code
from .metrics import FlopLedger
from .mv_refine import count_refine_flops

CABR_MIN_BLOCK = 16


class MissingKeyLabels(RuntimeError):
    def __init__(self, frame_index: int):
        super().__init__(f"frame {frame_index} was declared a key frame but no label map is available for it")
        self.frame_index = frame_index


@dataclass(frozen=True)
class RunResult:
    labels: list
    decisions: list
    ledger: FlopLedger
    scale: int

    @property
    def keyframes(self) -> int:
        return sum(d.kind is DecisionKind.KEY for d in self.decisions)


def _plane_geometry(frame: Frame, config: PipelineConfig):
    scale = mv_scale(frame)
    coarse = config.fme.block_sizes[0]
    return scale, -(-(frame.width // scale) // coarse), -(-(frame.height // scale) // coarse)


def _check_clip(frames) -> None:
    f0 = frames[0]
    for f in frames[1:]:
        if f.kind != f0.kind:
            raise ValueError(f"frame kind mismatch: {f.kind} vs {f0.kind}")
        if (f.width, f.height) != (f0.width, f0.height):
            raise ValueError("frame size mismatch")
        if f.data.dtype != f0.data.dtype:
            raise NotImplementedError("mixed uint8/uint16 clips are not supported by the B200 kernels")


def run_sequence(frames, key_labels, config: PipelineConfig = PipelineConfig(), weights=None) -> RunResult:
    """ME -> refine -> decide -> predict over an in-memory clip, on the GPU."""
    frames = list(frames)
    if not frames:
        raise ValueError("empty frame sequence")
    lookup = key_labels if callable(key_labels) else (lambda i: key_labels[i])
    scale, _, _ = _plane_geometry(frames[0], config)
    final_block = config.fme.block_sizes[-1] * scale
    if config.refine_enabled and final_block < CABR_MIN_BLOCK:
        raise ValueError(f"CaBR block size must be at least {CABR_MIN_BLOCK}: the finest FME level yields "
                         f"{final_block}-pixel blocks; disable refinement or use larger blocks")
    if config.refine_enabled:
        raise NotImplementedError("CaBR-Net block refinement is not part of the B200 hot path yet; "
                                  "run with PipelineConfig(refine_enabled=False)")
    _check_clip(frames)
    planes = 4 if scale == 2 else 1
    backbone = round(config.backbone_gflops * 1e9)

    f0 = frames[0]
    eng = ClipEngine(config, f0.height, f0.width, len(frames), 1, f0.data.dtype, f0.kind.is_bayer)
    eng.load_frames(np.stack([f.data for f in frames]))
    eng.motion()
    kinds, refs, trig = eng.decisions_host()
    kinds, refs, trig = kinds[0], refs[0], trig[0]

    injected = {}
    for i in range(len(frames)):
        if kinds[i] != 0:
            continue
        try:
            lab = lookup(i)
        except (KeyError, IndexError, FileNotFoundError):
            raise MissingKeyLabels(i) from None
        if lab is None:
            raise MissingKeyLabels(i)
        if not injected:
            eng.set_label_size(lab.height, lab.width)
        elif (lab.height, lab.width) != (eng.Hl, eng.Wl):
            raise ValueError("all key label maps of a clip must share one size")
        injected[i] = lab
        eng.key_labels[0, i].copy_(eng.torch.from_numpy(np.array(lab.classes)))
    eng.predict()
    out = eng.labels[0].cpu().numpy()

    ledger = FlopLedger()
    labels, decisions = [], []
    fin = eng.levels[-1]
    evals = [lv.evals[:eng.n_pairs].cpu().numpy() for lv in eng.levels]
    # count_replacements (mv_refine.py:72-73) counts changed vectors
    changed = (fin.mv[:eng.n_pairs] != eng.mv_ref[:eng.n_pairs]).any(dim=-1).sum(dim=(1, 2)).cpu().numpy()
    for i, f in enumerate(frames):
        if i > 0:
            p = eng.pair_index(0, i)
            ledger.add("fme", count_fme_flops((f.width, f.height), config.fme, [int(e[p]) for e in evals], planes))
            ledger.add("mv_refine", count_refine_flops(fin.gw, fin.gh, eng.b_final, int(changed[p]), planes))
        if kinds[i] == 0:
            ledger.add("backbone", backbone)
            lab = injected[i]
            decisions.append(FrameDecision(i, DecisionKind.KEY, None, float(trig[i])))
        else:
            ref = int(refs[i])
            lab = LabelMap(width=eng.Wl, height=eng.Hl, classes=out[i], num_classes=labels[ref].num_classes)
            ledger.add("prediction", 0)
            decisions.append(FrameDecision(i, kind_from_code(kinds[i]), ref, float(trig[i])))
        labels.append(lab)
    return RunResult(labels=labels, decisions=decisions, ledger=ledger, scale=scale)


class ClipSession:
    """Reusable host-buffer clip API (the batched public entry point).

    ``run(raw, key_labels)`` takes a (T, H, W) uint8/uint16 Bayer (or luma)
    clip in host memory, runs ME -> refine -> decide -> predict on the GPU and
    returns ``(labels (T, Hl, Wl) uint8 ndarray, kinds, refs, triggers)``.
    ``key_labels`` is a callable / mapping frame -> LabelMap consulted exactly
    once per key frame, as in ``run_sequence``.  Device buffers and pinned
    staging buffers are allocated once per session, so repeated clips of the
    same geometry pay only the transfers and the kernels.
    """

    def __init__(self, config: PipelineConfig, height: int, width: int, n_frames: int, dtype=np.uint8,
                 bayer: bool = True):
        if config.refine_enabled:
            raise NotImplementedError("CaBR-Net block refinement is not part of the B200 hot path yet; "
                                      "run with PipelineConfig(refine_enabled=False)")
        self.eng = ClipEngine(config, height, width, n_frames, 1, dtype, bayer)
        torch = self.eng.torch
        self.torch = torch
        self.pin_raw = torch.empty(tuple(self.eng.raw.shape[1:]), dtype=self.eng.raw.dtype).pin_memory()
        self.pin_labels = torch.empty(tuple(self.eng.labels.shape[1:]), dtype=torch.uint8).pin_memory()
        self.pin_key = torch.empty(tuple(self.eng.labels.shape[1:]), dtype=torch.uint8).pin_memory()
        self.h2d_bytes = 0
        self.d2h_bytes = 0

    def run(self, raw, key_labels):
        eng, torch = self.eng, self.torch
        lookup = key_labels if callable(key_labels) else (lambda i: key_labels[i])
        src = raw if isinstance(raw, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(raw))
        if src.is_pinned():
            eng.raw[0].copy_(src, non_blocking=True)
        else:
            self.pin_raw.copy_(src)
            eng.raw[0].copy_(self.pin_raw, non_blocking=True)
        h2d = src.numel() * src.element_size()
        eng.motion()
        kinds, refs, trig = (a[0] for a in eng.decisions_host())
        d2h = kinds.nbytes + refs.nbytes + trig.nbytes
        for i in np.nonzero(kinds == 0)[0].tolist():
            try:
                lab = lookup(i)
            except (KeyError, IndexError, FileNotFoundError):
                raise MissingKeyLabels(i) from None
            if lab is None:
                raise MissingKeyLabels(i)
            if (lab.height, lab.width) != (eng.Hl, eng.Wl):
                raise ValueError("key label maps must match the session's label size")
            self.pin_key[i].copy_(torch.from_numpy(np.array(lab.classes)))
            eng.key_labels[0, i].copy_(self.pin_key[i], non_blocking=True)
            h2d += lab.classes.nbytes
        eng.predict()
        self.pin_labels.copy_(eng.labels[0], non_blocking=True)
        torch.cuda.current_stream().synchronize()
        d2h += self.pin_labels.numel()
        self.h2d_bytes, self.d2h_bytes = h2d, d2h
        return self.pin_labels.numpy(), kinds, refs, trig
