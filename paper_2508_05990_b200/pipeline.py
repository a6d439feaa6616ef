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
kernel does the same on device.  With ``weights`` the CaBR-Net forward pass
re-labels them instead (``bmc_cabr_chain``: per predicted frame, prediction,
the network over the frame's flagged blocks, write-back).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .config import PipelineConfig
from .cabr import count_cabr_flops
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
    use_net = config.refine_enabled and weights is not None
    flagged = np.zeros(len(frames), dtype=np.int64)  # refinement_blocks per predicted frame
    if use_net and len(frames) > 1:
        m = eng.levels[-1].matched[:eng.n_pairs].cpu().numpy()
        for i in range(1, len(frames)):
            if kinds[i] != 0:
                flagged[i] = int((m[eng.pair_index(0, i)] == 0).sum())
    if use_net and flagged.any():
        C = next(iter(injected.values())).num_classes
        if weights.num_classes != C:
            raise ValueError("weights and label map disagree on num_classes")
        eng.set_cabr(weights)
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
            if use_net:
                ledger.add("cabr", count_cabr_flops(eng.b_final * scale, labels[ref].num_classes, int(flagged[i])))
            decisions.append(FrameDecision(i, kind_from_code(kinds[i]), ref, float(trig[i])))
        labels.append(lab)
    return RunResult(labels=labels, decisions=decisions, ledger=ledger, scale=scale)


class ClipSession:
    """Reusable host-buffer clip API (the batched public entry point).

    ``run(raw, key_labels)`` takes a (T, H, W) uint8/uint16 Bayer (or luma)
    clip in host memory, runs ME -> refine -> decide -> predict on the GPU and
    returns ``(labels, kinds, refs, triggers)`` where ``labels`` is a list of T
    (Hl, Wl) uint8 arrays.

    ``key_labels`` is either
      * a callable / mapping frame -> LabelMap consulted exactly once per key
        frame, in frame order, as ``run_sequence`` does, or
      * a (T, Hl, Wl) uint8 tensor (pinned for full speed) holding a label map
        for every frame; only the key frames' maps are used (reference
        semantics).

    ``weights`` (CabrWeights) runs the CaBR-Net forward pass on the flagged
    blocks of predicted frames, as ``run_sequence(..., weights)`` does.

    Data movement follows the reference's semantics rather than shipping whole
    label stacks: a key frame's output IS its input label map
    (pipeline.py:116-121 appends the injected LabelMap), so it is returned as
    that host array and never copied back; a key map is uploaded only when a
    predicted frame references it; only predicted frames' labels come back.

    With the default "previous" reference policy the clip is processed in
    ``chunks`` frame ranges, software-pipelined by ``lag`` chunks on three
    streams: the H2D of chunk c+lag's raw frames, pack, ME, refine and the AEM
    scan are queued before the host reads chunk c's decisions (by then long
    finished), so the GPU never waits for the host; chunk c's needed key maps
    are then uploaded, its label chain runs and its predicted labels stream
    back while later chunks compute.  Results are identical to ``run_sequence`` (chunking
    only changes launch boundaries).  Returned arrays owned by the session are
    overwritten by the next ``run``.
    """

    def __init__(self, config: PipelineConfig, height: int, width: int, n_frames: int, dtype=np.uint8,
                 bayer: bool = True, chunks: int = 5, lag: int = 2, weights=None, ramp: float = 1.0):
        if config.refine_enabled and config.fme.block_sizes[-1] * (2 if bayer else 1) < CABR_MIN_BLOCK:
            raise ValueError(f"CaBR block size must be at least {CABR_MIN_BLOCK}: the finest FME level yields "
                             f"{config.fme.block_sizes[-1] * (2 if bayer else 1)}-pixel blocks; disable refinement "
                             f"or use larger blocks")
        self.eng = ClipEngine(config, height, width, n_frames, 1, dtype, bayer)
        if weights is not None and config.refine_enabled:  # CaBR-Net instead of the ring vote
            self.eng.set_cabr(weights)
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
        # chunk c ends at t * ((c+1)/k)^ramp: ramp > 1 makes the first chunks short, so
        # the GPU starts after a small H2D while later (longer) copies overlap compute
        bounds = [round(t * (i / k) ** float(ramp)) for i in range(k + 1)]
        self.chunks = [(bounds[i], bounds[i + 1]) for i in range(k) if bounds[i + 1] > bounds[i]]
        self.lag = max(1, int(lag))
        self.h2d_bytes = 0
        self.d2h_bytes = 0
        self._native = self._native_session() if (config.reference_policy == "previous" and t >= 2
                                                  and len(self.chunks) <= N.Session.MAX_CHUNKS) else None

    def _native_session(self):
        """bmc_session over this session's device and pinned buffers (include/bmc_ext.h): the
        chunk schedule of run() for key maps given as one tensor, executed natively."""
        eng, torch = self.eng, self.torch
        s = N.Session()
        s.T, s.H, s.W = eng.T, eng.H, eng.W
        s.elem_bytes, s.kind = eng.raw.element_size(), eng.kind_code
        s.n_chunks, s.lag = len(self.chunks), self.lag
        for k, (f0, _f1) in enumerate(self.chunks):
            s.chunk_begin[k] = f0
        s.chunk_begin[len(self.chunks)] = self.chunks[-1][1]
        s.gh, s.gw, s.b_final, s.scale = eng.gh, eng.gw, eng.b_final, eng.scale
        s.deviation_threshold = int(eng.cfg.deviation_threshold)
        s.n_levels, s.Hl, s.Wl, s.ring_vote = len(eng.levels), eng.Hl, eng.Wl, int(eng.ring_vote)
        s.params, s.select = eng.params, eng.sp
        s.raw, s.planes = N.ptr(eng.raw), N.ptr(eng.planes)
        s.cur_index, s.ref_index = N.ptr(eng.cur_index), N.ptr(eng.ref_index)
        for k, lv in enumerate(eng.levels):
            s.levels[k] = N.LevelOut(N.ptr(lv.mv), N.ptr(lv.energy), N.ptr(lv.matched), N.ptr(lv.evals))
        s.mv_ref, s.e_ref, s.replaced = N.ptr(eng.mv_ref), N.ptr(eng.e_ref), N.ptr(eng.replaced)
        s.aem_state, s.aem_state_bytes = N.ptr(eng._aem_zero), eng._aem_zero.numel()
        s.acc, s.fsk, s.last_key = N.ptr(eng.acc), N.ptr(eng.fsk), N.ptr(eng.last_key)
        s.kind_out, s.ref_out, s.trigger = N.ptr(eng.kind), N.ptr(eng.ref), N.ptr(eng.trigger)
        s.labels, s.key_labels, s.chain_ws = N.ptr(eng.labels), N.ptr(eng.key_labels), N.ptr(eng.workspace)
        if eng.cabr is not None:
            c = eng.cabr
            s.cabr_packed, s.cabr_classes = N.ptr(c["packed"]), c["C"]
            s.cabr_scratch, s.cabr_ws = N.ptr(c["scratch"]), N.ptr(c["workspace"])
        self.host_kind = torch.empty(eng.T, dtype=torch.int32).pin_memory()
        self.host_ref = torch.empty(eng.T, dtype=torch.int32).pin_memory()
        self.host_trigger = torch.empty(eng.T, dtype=torch.float64).pin_memory()
        s.host_labels = N.ptr(self.pin_labels)
        s.host_kind, s.host_ref, s.host_trigger = N.ptr(self.host_kind), N.ptr(self.host_ref), N.ptr(self.host_trigger)
        s.copy_in, s.copy_out = N.stream_handle(self.copy_in), N.stream_handle(self.copy_out)
        N.check(N.load().bmc_session_init(ctypes.byref(s)))
        self._pin_labels_np = self.pin_labels.numpy()
        return s

    def __del__(self):
        s = getattr(self, "_native", None)
        if s is not None and s.priv:
            try:
                N.load().bmc_session_destroy(ctypes.byref(s))
            except Exception:  # interpreter shutdown: module globals already cleared
                pass

    def _run_native(self, src, keys):
        """One clip through bmc_session_run (key maps as one pinned (T, Hl, Wl) tensor)."""
        eng, torch = self.eng, self.torch
        if not (keys.is_pinned() and keys.is_contiguous() and keys.dtype == torch.uint8):
            self.pin_key.copy_(keys)
            keys = self.pin_key
        s = self._native
        s.host_raw, s.host_keys = src.data_ptr(), keys.data_ptr()
        s.compute = N.stream_handle()
        N.check(N.load().bmc_session_run(ctypes.byref(s)))
        kinds, refs = self.host_kind.numpy().copy(), self.host_ref.numpy().copy()
        trig = self.host_trigger.numpy().copy()
        keys_np, pred_np = keys.numpy(), self._pin_labels_np
        labels = [keys_np[i] if kinds[i] == 0 else pred_np[i] for i in range(eng.T)]
        self.h2d_bytes, self.d2h_bytes = int(s.h2d_bytes), int(s.d2h_bytes)
        return labels, kinds, refs, trig

    # -- helpers ----------------------------------------------------------------
    def _motion_chunk(self, src, f0: int, f1: int) -> None:
        """H2D of frames [f0, f1) (copy stream), then pack, ME of the pairs whose frames
        are resident, refine and the AEM scan of those frames (compute stream)."""
        eng, torch = self.eng, self.torch
        lib = N.load()
        cs = torch.cuda.current_stream()
        st = N.stream_handle(cs)
        p = eng.params
        ev = torch.cuda.Event()
        with torch.cuda.stream(self.copy_in):
            eng.raw[0, f0:f1].copy_(src[f0:f1], non_blocking=True)
            ev.record(self.copy_in)
        cs.wait_event(ev)
        N.check(lib.bmc_pack_planes(N.ptr(eng.raw[0, f0]), f1 - f0, eng.kind_code, ctypes.byref(p),
                                    N.ptr(eng.planes) + f0 * p.frame_stride * eng.planes.element_size(), st))
        p0, p1 = max(f0, 1) - 1, f1 - 1  # pairs t in [max(f0,1), f1): both frames resident
        if p1 > p0:
            arr = eng._level_slice(p0, p1)
            N.check(lib.bmc_estimate_motion(N.ptr(eng.planes), eng.S * eng.T, ctypes.byref(p), p1 - p0,
                                            N.ptr(eng.cur_index[p0:p1]), N.ptr(eng.ref_index[p0:p1]), arr, st))
            eng._refine(p0, p1)
            eng._decide(p0 + 1, p1 + 1)

    def _decisions_out(self, f0: int, f1: int):
        """D2H of frames [f0, f1)'s decisions (copy-out stream, after the compute stream's AEM scan)."""
        eng, torch = self.eng, self.torch
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream())
        with torch.cuda.stream(self.copy_out):
            self.copy_out.wait_event(ev)
            self.pin_dec[0, f0:f1].copy_(eng.kind[0, f0:f1], non_blocking=True)
            self.pin_dec[1, f0:f1].copy_(eng.ref[0, f0:f1], non_blocking=True)
            self.pin_dec[2, f0:f1].copy_(eng.trigger[0, f0:f1], non_blocking=True)
            done = torch.cuda.Event()
            done.record(self.copy_out)
        return done

    def _finish_chunk(self, f0: int, f1: int, dec_done, state) -> None:
        """Host reads frames [f0, f1)'s decisions, consults the key labels, uploads the key
        maps predicted frames reference, runs the chunk's label chain and streams the
        predicted frames' labels back."""
        eng, torch = self.eng, self.torch
        dec_done.synchronize()
        kinds = self.pin_dec[0, f0:f1].numpy().astype(np.int32)
        refs = self.pin_dec[1, f0:f1].numpy().astype(np.int32)
        all_kinds = state["kinds"]
        all_kinds[f0:f1] = kinds
        for i in range(f0, f1):
            if kinds[i - f0] == 0:
                state["key_host"][i] = self._key_map(state, i)
        need = sorted({int(r) for k, r in zip(kinds, refs) if k != 0 and all_kinds[int(r)] == 0}
                      - state["uploaded"])
        cs = torch.cuda.current_stream()
        if need:
            ev = torch.cuda.Event()
            with torch.cuda.stream(self.copy_in):
                if state["chain_done"] is not None and min(need) < f0:
                    # labels[r] of an earlier chunk's key frame: that chunk's chain (compute
                    # stream) wrote its slot from key_labels, so the upload must land after it
                    self.copy_in.wait_event(state["chain_done"])
                for r in need:
                    # a key in this chunk goes to key_labels (its chain copies it into labels);
                    # one in an earlier chunk was already chained, so it goes straight to labels
                    dst = eng.key_labels[0, r] if r >= f0 else eng.labels[0, r]
                    host = state["key_host"][r]
                    if isinstance(host, torch.Tensor) and host.is_pinned():
                        dst.copy_(host, non_blocking=True)
                    else:
                        self.pin_key[r].numpy()[...] = host
                        dst.copy_(self.pin_key[r], non_blocking=True)
                    state["h2d"] += eng.Hl * eng.Wl
                ev.record(self.copy_in)
            cs.wait_event(ev)
            state["uploaded"].update(need)
        eng._chain(f0, f1)
        state["chain_done"] = torch.cuda.Event()
        state["chain_done"].record(cs)
        pred = [i for i in range(f0, f1) if kinds[i - f0] != 0]
        if pred:
            ev = torch.cuda.Event()
            ev.record(cs)
            with torch.cuda.stream(self.copy_out):
                self.copy_out.wait_event(ev)
                i = 0
                while i < len(pred):  # runs of consecutive predicted frames, one copy each
                    j = i
                    while j + 1 < len(pred) and pred[j + 1] == pred[j] + 1:
                        j += 1
                    self.pin_labels[pred[i]:pred[j] + 1].copy_(eng.labels[0, pred[i]:pred[j] + 1], non_blocking=True)
                    state["d2h"] += (pred[j] + 1 - pred[i]) * eng.Hl * eng.Wl
                    i = j + 1

    def _key_map(self, state, i: int):
        """Key frame i's label map as a host array/tensor (the reference's lookup, in frame order)."""
        eng = self.eng
        tensor = state["tensor"]
        if tensor is not None:
            return tensor[i]
        try:
            lab = state["lookup"](i)
        except (KeyError, IndexError, FileNotFoundError):
            raise MissingKeyLabels(i) from None
        if lab is None:
            raise MissingKeyLabels(i)
        if (lab.height, lab.width) != (eng.Hl, eng.Wl):
            raise ValueError("key label maps must match the session's label size")
        return lab.classes

    def run(self, raw, key_labels):
        eng, torch = self.eng, self.torch
        src = raw if isinstance(raw, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(raw))
        if not src.is_pinned():
            self.pin_raw.copy_(src)
            src = self.pin_raw
        tensor = key_labels if isinstance(key_labels, torch.Tensor) else None
        if tensor is not None and tuple(tensor.shape) != tuple(eng.labels.shape[1:]):
            raise ValueError(f"key label tensor must be {tuple(eng.labels.shape[1:])}, got {tuple(tensor.shape)}")
        if tensor is not None and self._native is not None:
            return self._run_native(src, tensor)
        lookup = None
        if tensor is None:
            lookup = key_labels if callable(key_labels) else (lambda i: key_labels[i])
        state = {"tensor": tensor, "lookup": lookup, "kinds": np.full(eng.T, -1, np.int32), "key_host": {},
                 "uploaded": set(), "h2d": src.numel() * src.element_size(), "d2h": 0, "chain_done": None}
        self.copy_in.wait_stream(torch.cuda.current_stream())  # earlier users of the device buffers are done
        eng._reset_state()
        if eng.cfg.reference_policy == "previous" and eng.T >= 2:
            pending = []
            for f0, f1 in self.chunks:
                self._motion_chunk(src, f0, f1)
                pending.append((f0, f1, self._decisions_out(f0, f1)))
                if len(pending) > self.lag:  # the GPU keeps `lag` chunks of motion work queued
                    self._finish_chunk(*pending.pop(0), state)
            for item in pending:
                self._finish_chunk(*item, state)
        else:  # "keyframe" policy (each ME's reference comes from the previous decision) or T == 1
            ev = torch.cuda.Event()
            with torch.cuda.stream(self.copy_in):
                eng.raw[0].copy_(src, non_blocking=True)
                ev.record(self.copy_in)
            torch.cuda.current_stream().wait_event(ev)
            eng.motion()  # pack, reset, per-frame ME -> refine -> decide with device-chosen references
            done = self._decisions_out(0, eng.T)
            self._finish_chunk(0, eng.T, done, state)
        self.copy_out.synchronize()
        state["d2h"] += self.pin_dec.numel() * 8
        kinds = self.pin_dec[0].numpy().astype(np.int32)
        refs = self.pin_dec[1].numpy().astype(np.int32)
        trig = self.pin_dec[2].numpy().copy()
        labels = []
        for i in range(eng.T):
            if kinds[i] == 0:
                h = state["key_host"][i]
                labels.append(h.numpy() if isinstance(h, torch.Tensor) else np.asarray(h))
            else:
                labels.append(self.pin_labels[i].numpy())
        self.h2d_bytes, self.d2h_bytes = state["h2d"], state["d2h"]
        return labels, kinds, refs, trig


class ClipPool:
    """Many independent clips (streams) through ``n_sessions`` ClipSessions at once.

    Each session owns its device buffers and runs on its own compute stream; a
    host thread per session drives it (the native executor releases the GIL), so
    one clip's H2D, compute and D2H overlap another's -- the batched form of
    ``ClipSession.run`` for stream-parallel serving.
    ``run(clips)`` takes a list of ``(raw, key_labels)`` pairs (as
    ``ClipSession.run``) and returns their results in order.  Predicted frames'
    labels are copied out of the session buffers (a session's next clip
    overwrites them); key frames are returned as the caller's key maps.
    """

    def __init__(self, config: PipelineConfig, height: int, width: int, n_frames: int, dtype=np.uint8,
                 bayer: bool = True, n_sessions: int = 2, weights=None, **session_kw):
        import threading
        from concurrent.futures import ThreadPoolExecutor
        self.sessions = [ClipSession(config, height, width, n_frames, dtype, bayer, weights=weights, **session_kw)
                         for _ in range(max(1, int(n_sessions)))]
        torch = self.sessions[0].torch
        self.torch = torch
        self.streams = [torch.cuda.Stream() for _ in self.sessions]
        self.pool = ThreadPoolExecutor(max_workers=len(self.sessions))
        self.device = torch.cuda.current_device()
        self._lock = threading.Lock()
        self.h2d_bytes = 0
        self.d2h_bytes = 0

    def _worker(self, k, items):
        torch = self.torch
        torch.cuda.set_device(self.device)
        sess, st = self.sessions[k], self.streams[k]
        out, h2d, d2h = [], 0, 0
        with torch.cuda.stream(st):
            for idx, (raw, keys) in items:
                labels, kinds, refs, trig = sess.run(raw, keys)
                # predicted frames live in the session's output buffer (overwritten by its next
                # clip): copy those; key frames are the caller's own key maps
                labels = [np.array(x) if kinds[i] != 0 else x for i, x in enumerate(labels)]
                out.append((idx, (labels, kinds, refs, trig)))
                h2d += sess.h2d_bytes
                d2h += sess.d2h_bytes
        return out, h2d, d2h

    def run(self, clips):
        torch = self.torch
        cur = torch.cuda.current_stream()
        for st in self.streams:  # earlier work of the caller's stream is visible to every session
            st.wait_stream(cur)
        n = len(self.sessions)
        parts = [[(i, c) for i, c in enumerate(clips) if i % n == k] for k in range(n)]
        futs = [self.pool.submit(self._worker, k, parts[k]) for k in range(n)]
        results = [None] * len(clips)
        self.h2d_bytes = self.d2h_bytes = 0
        for f in futs:
            out, h2d, d2h = f.result()
            self.h2d_bytes += h2d
            self.d2h_bytes += d2h
            for idx, r in out:
                results[idx] = r
        for st in self.streams:
            cur.wait_stream(st)
        return results
