"""Sequence driver (drop-in for ``bayermc.pipeline.run_sequence``, pipeline.py:23-141).

The reference walks frames one by one on the CPU.  Here the whole clip runs
in a ``ClipEngine`` on the GPU in two device passes separated by ONE host
round trip:

  1. motion pass: pack, ME, MV refinement and the AEM scan for every frame;
  2. the host reads the decisions, asks ``key_labels`` for exactly the key
     frames (in frame order, as the reference does), uploads them, and
  3. prediction pass: the label chain on device.

Semantics (decisions, labels, ledger) are identical to the reference's.  With
``refine_enabled`` (the default) and no CaBR weights the reference re-labels the
flagged blocks of every predicted frame with its weight-free ring vote
(cabr.py:257-345) and the refined labels feed later predictions; the label-chain
kernel does the same on device.  Running the CaBR-Net forward pass itself
(``weights`` given) is the next component on the roadmap and raises instead of
silently skipping it.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native as N
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
    if config.refine_enabled and weights is not None:
        raise NotImplementedError("the CaBR-Net forward pass (weights given) is not part of the B200 hot path yet; "
                                  "pass weights=None for the ring-vote fallback or disable refinement")
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

    ``key_labels`` is either
      * a callable / mapping frame -> LabelMap consulted exactly once per key
        frame, in frame order, as ``run_sequence`` does (decisions are read back
        first, then the key frames' labels are uploaded), or
      * a (T, Hl, Wl) uint8 tensor (pinned for full speed) holding a label map
        for every frame; only the key frames' maps are used (reference
        semantics), and the upload overlaps motion estimation.

    With the default "previous" reference policy the clip is processed in
    ``chunks`` frame ranges on three streams: the H2D copy of chunk c+1
    overlaps pack + ME of chunk c; refine and the AEM scan follow; the label
    chain then runs per chunk with each chunk's D2H overlapping the next
    chunk's gathers.  Results are identical to ``run_sequence`` (the chunking
    only changes launch boundaries).  The returned label array is owned by the
    session and overwritten by the next ``run``.
    """

    def __init__(self, config: PipelineConfig, height: int, width: int, n_frames: int, dtype=np.uint8,
                 bayer: bool = True, chunks: int = 10):
        if config.refine_enabled and config.fme.block_sizes[-1] * (2 if bayer else 1) < CABR_MIN_BLOCK:
            raise ValueError(f"CaBR block size must be at least {CABR_MIN_BLOCK}: the finest FME level yields "
                             f"{config.fme.block_sizes[-1] * (2 if bayer else 1)}-pixel blocks; disable refinement "
                             f"or use larger blocks")
        self.eng = ClipEngine(config, height, width, n_frames, 1, dtype, bayer)
        torch = self.eng.torch
        self.torch = torch
        self.pin_raw = torch.empty(tuple(self.eng.raw.shape[1:]), dtype=self.eng.raw.dtype).pin_memory()
        self.pin_labels = torch.empty(tuple(self.eng.labels.shape[1:]), dtype=torch.uint8).pin_memory()
        self.pin_key = torch.empty(tuple(self.eng.labels.shape[1:]), dtype=torch.uint8).pin_memory()
        self.pin_dec = torch.empty((3, n_frames), dtype=torch.float64).pin_memory()
        self.copy_in = torch.cuda.Stream()
        self.copy_out = torch.cuda.Stream()
        t = int(n_frames)
        k = max(1, min(int(chunks), t))
        bounds = [round(i * t / k) for i in range(k + 1)]
        self.chunks = [(bounds[i], bounds[i + 1]) for i in range(k) if bounds[i + 1] > bounds[i]]
        self.h2d_bytes = 0
        self.d2h_bytes = 0

    # -- helpers ----------------------------------------------------------------
    def _lookup_keys(self, lookup, kinds):
        eng, torch = self.eng, self.torch
        h2d = 0
        for i in np.nonzero(kinds == 0)[0].tolist():
            try:
                lab = lookup(i)
            except (KeyError, IndexError, FileNotFoundError):
                raise MissingKeyLabels(i) from None
            if lab is None:
                raise MissingKeyLabels(i)
            if (lab.height, lab.width) != (eng.Hl, eng.Wl):
                raise ValueError("key label maps must match the session's label size")
            np.copyto(self.pin_key[i].numpy(), lab.classes)
            eng.key_labels[0, i].copy_(self.pin_key[i], non_blocking=True)
            h2d += lab.classes.nbytes
        return h2d

    def _run_streamed(self, src, label_tensor, h2d):
        """Fully chunked pass ("previous" policy, labels as a tensor): per frame chunk
        H2D (raw + label maps) -> pack -> ME -> refine -> AEM scan (resumable state)
        -> label chain -> D2H, so copies in both directions overlap the kernels of
        neighbouring chunks.  Every step only needs frames of its own or earlier
        chunks (pair t uses frames t-1, t; the AEM scan and the label chain are
        causal), so results equal the whole-clip pass."""
        eng, torch = self.eng, self.torch
        lib = N.load()
        cs = torch.cuda.current_stream()
        st = N.stream_handle(cs)
        p = eng.params
        fstride = p.frame_stride
        esz = eng.planes.element_size()
        cells2 = eng.gh * eng.gw * 2
        fs = eng.Hl * eng.Wl
        eng._reset_state()
        self.copy_in.wait_stream(cs)  # previous users of the input buffers are done
        for f0, f1 in self.chunks:
            ev_in = torch.cuda.Event()
            with torch.cuda.stream(self.copy_in):
                eng.raw[0, f0:f1].copy_(src[f0:f1], non_blocking=True)
                eng.key_labels[0, f0:f1].copy_(label_tensor[f0:f1], non_blocking=True)
                ev_in.record(self.copy_in)
            cs.wait_event(ev_in)
            N.check(lib.bmc_pack_planes(N.ptr(eng.raw[0, f0]), f1 - f0, eng.kind_code, ctypes.byref(p),
                                        N.ptr(eng.planes) + f0 * fstride * esz, st))
            p0, p1 = max(f0, 1) - 1, f1 - 1
            if p1 > p0:
                arr = eng._level_slice(p0, p1)
                N.check(lib.bmc_estimate_motion(N.ptr(eng.planes), eng.S * eng.T, ctypes.byref(p), p1 - p0,
                                                N.ptr(eng.cur_index[p0:p1]), N.ptr(eng.ref_index[p0:p1]), arr, st))
                eng._refine(p0, p1)
                eng._decide(p0 + 1, p1 + 1)
            eng._chain(f0, f1)
            ev_out = torch.cuda.Event()
            ev_out.record(cs)
            with torch.cuda.stream(self.copy_out):
                self.copy_out.wait_event(ev_out)
                self.pin_labels[f0:f1].copy_(eng.labels[0, f0:f1], non_blocking=True)
        dec = torch.stack([eng.kind[0].double(), eng.ref[0].double(), eng.trigger[0]])
        ev = torch.cuda.Event()
        ev.record(cs)
        with torch.cuda.stream(self.copy_out):
            self.copy_out.wait_event(ev)
            self.pin_dec.copy_(dec, non_blocking=True)
        self.copy_out.synchronize()
        kinds = self.pin_dec[0].numpy().astype(np.int32)
        refs = self.pin_dec[1].numpy().astype(np.int32)
        trig = self.pin_dec[2].numpy().copy()
        self.h2d_bytes = h2d + label_tensor.numel()
        self.d2h_bytes = self.pin_dec.numel() * 8 + self.pin_labels.numel()
        return self.pin_labels.numpy(), kinds, refs, trig

    def run(self, raw, key_labels):
        eng, torch = self.eng, self.torch
        lib = N.load()
        cs = torch.cuda.current_stream()
        st = N.stream_handle(cs)
        src = raw if isinstance(raw, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(raw))
        if not src.is_pinned():
            self.pin_raw.copy_(src)
            src = self.pin_raw
        label_tensor = key_labels if isinstance(key_labels, torch.Tensor) else None
        lookup = None
        if label_tensor is None:
            lookup = key_labels if callable(key_labels) else (lambda i: key_labels[i])
        elif tuple(label_tensor.shape) != tuple(eng.labels.shape[1:]):
            raise ValueError(f"key label tensor must be {tuple(eng.labels.shape[1:])}, got {tuple(label_tensor.shape)}")
        h2d = src.numel() * src.element_size()
        p = eng.params
        fstride = p.frame_stride
        esz = eng.planes.element_size()
        eng._reset_state()
        pipelined = eng.cfg.reference_policy == "previous" and eng.T >= 2
        if pipelined and label_tensor is not None:
            return self._run_streamed(src, label_tensor, h2d)
        if pipelined:
            for f0, f1 in self.chunks:
                ev = torch.cuda.Event()
                with torch.cuda.stream(self.copy_in):
                    self.copy_in.wait_stream(cs)  # previous users of eng.raw are done
                    eng.raw[0, f0:f1].copy_(src[f0:f1], non_blocking=True)
                    ev.record(self.copy_in)
                cs.wait_event(ev)
                N.check(lib.bmc_pack_planes(N.ptr(eng.raw[0, f0]), f1 - f0, eng.kind_code, ctypes.byref(p),
                                            N.ptr(eng.planes) + f0 * fstride * esz, st))
                p0, p1 = max(f0, 1) - 1, f1 - 1  # pairs whose frames are resident: t in [max(f0,1), f1)
                if p1 > p0:
                    arr = eng._level_slice(p0, p1)
                    N.check(lib.bmc_estimate_motion(N.ptr(eng.planes), eng.S * eng.T, ctypes.byref(p), p1 - p0,
                                                    N.ptr(eng.cur_index[p0:p1]), N.ptr(eng.ref_index[p0:p1]), arr, st))
            if label_tensor is not None:
                ev_lab = torch.cuda.Event()
                with torch.cuda.stream(self.copy_in):
                    eng.key_labels[0].copy_(label_tensor, non_blocking=True)
                    ev_lab.record(self.copy_in)
            eng._refine(0, eng.n_pairs)
            eng._decide(1, eng.T)
        else:
            eng.raw[0].copy_(src, non_blocking=True)
            eng.motion()
            if label_tensor is not None:
                eng.key_labels[0].copy_(label_tensor, non_blocking=True)
        dec = torch.stack([eng.kind[0].double(), eng.ref[0].double(), eng.trigger[0]])
        d2h = self.pin_dec.numel() * 8  # kind, ref, trigger (float64 rows)
        if label_tensor is None:
            self.pin_dec.copy_(dec)  # synchronous: the key lookups need the decisions
            kinds = self.pin_dec[0].numpy().astype(np.int32)
            h2d += self._lookup_keys(lookup, kinds)
        else:
            if pipelined:
                cs.wait_event(ev_lab)
            h2d += label_tensor.numel()  # whole tensor uploaded (every frame's map is an input)
        # label chain per chunk; each chunk's D2H overlaps the next chunk's gathers
        cells2 = eng.gh * eng.gw * 2
        fs = eng.Hl * eng.Wl
        chunks = self.chunks if pipelined else [(0, eng.T)]
        for f0, f1 in chunks:
            eng._chain(f0, f1)
            ev = torch.cuda.Event()
            ev.record(cs)
            with torch.cuda.stream(self.copy_out):
                self.copy_out.wait_event(ev)
                self.pin_labels[f0:f1].copy_(eng.labels[0, f0:f1], non_blocking=True)
        if label_tensor is not None:
            with torch.cuda.stream(self.copy_out):
                self.pin_dec.copy_(dec, non_blocking=True)
        self.copy_out.synchronize()
        kinds = self.pin_dec[0].numpy().astype(np.int32)
        refs = self.pin_dec[1].numpy().astype(np.int32)
        trig = self.pin_dec[2].numpy().copy()
        d2h += self.pin_labels.numel()
        self.h2d_bytes, self.d2h_bytes = h2d, d2h
        return self.pin_labels.numpy(), kinds, refs, trig
