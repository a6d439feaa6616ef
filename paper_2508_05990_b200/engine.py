"""Device-resident batched pipeline: S streams x T frames per step.

This is the B200 replacement of the per-frame loop in ``run_sequence``
(pipeline.py:97-141) minus CaBR.  One step is

  pack (raw Bayer -> padded CFA planes)            bmc_pack_planes
  ME for every frame pair, all levels              bmc_estimate_motion
  3x3 MV refinement + energy re-evaluation         bmc_refine_mvs
  AEM key-frame scan over the clip                 bmc_decide
  label propagation chain (key copy / gather)      bmc_predict_labels_clip (one cooperative launch)

all enqueued on one CUDA stream with no host synchronisation, so the whole
step can be captured in a CUDA graph.  With the default "previous" reference
policy ME/refine of all pairs of all streams run as ONE launch each (the pairs
are independent); with "keyframe" the reference frame depends on earlier
decisions, so ME/refine/decide run frame by frame, with the decide kernel
writing the next frame's reference index straight into the ME index array.

Device layouts (pair p of frame t >= 1 of stream s is p = (t-1)*S + s):
  raw        (S, T, H, W)           uint8/uint16
  planes     (S*T, P, pad_h, pitch) uint8/uint16
  levels[L]  mv (pairs, gh, gw, 2) int32, energy f64, matched u8, evals i64
  refined    mv (pairs, gh, gw, 2) int32, energy f64
  decisions  kind/ref (S, T) int32, trigger (S, T) f64
  labels     (S, T, Hl, Wl) uint8 (key_labels: same layout, key slots used)
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _device as D
from . import _native as N
from .config import PipelineConfig


class ClipEngine:
    def __init__(self, config: PipelineConfig, height: int, width: int, n_frames: int, n_streams: int = 1,
                 dtype=np.uint8, bayer: bool = True, label_hw=None):
        torch = N.require_cuda()
        if config.aem_statistic not in ("max", "mean"):
            raise ValueError("statistic must be 'max' or 'mean'")
        if config.reference_policy not in ("previous", "keyframe"):
            raise ValueError("reference_policy must be 'previous' or 'keyframe'")
        if n_frames < 1 or n_streams < 1:
            raise ValueError("need at least one frame and one stream")
        if any(b > 64 for b in config.fme.block_sizes):
            raise NotImplementedError(
                f"the clip engine's integer search kernels take block sizes 8..64, got {config.fme.block_sizes}; "
                "fme.estimate_motion / search_stage / refine_mvs accept larger blocks (float64 kernel)")
        self.torch = torch
        self.cfg = config
        self.S, self.T, self.H, self.W = int(n_streams), int(n_frames), int(height), int(width)
        self.bayer = bool(bayer)
        self.scale = 2 if self.bayer else 1
        tdt = torch.uint8 if np.dtype(dtype) == np.uint8 else torch.uint16
        self.dev = torch.device("cuda", torch.cuda.current_device())
        self.kind_code = N.KIND_BAYER if self.bayer else N.KIND_LUMA
        self.params = N.make_params(self.kind_code, 1 if tdt == torch.uint8 else 2, self.H, self.W, config.fme)
        p = self.params
        lib = N.load()
        S, T = self.S, self.T
        self.raw = torch.zeros((S, T, self.H, self.W), dtype=tdt, device=self.dev)
        self.planes = torch.empty(lib.bmc_plane_buffer_elems(ctypes.byref(p), S * T), dtype=tdt, device=self.dev)
        self.n_pairs = S * (T - 1)
        t = torch.arange(1, T, dtype=torch.int32, device=self.dev).repeat_interleave(S)
        s = torch.arange(S, dtype=torch.int32, device=self.dev).repeat(T - 1)
        self.cur_index = (s * T + t).contiguous()
        self.ref_index_init = (s * T + t - 1).contiguous() if config.reference_policy == "previous" \
            else (s * T).contiguous()
        self.ref_index = self.ref_index_init.clone()
        sizes = list(config.fme.block_sizes)
        self.levels = [D.LevelBuffers(torch, self.dev, max(self.n_pairs, 1), p.pad_h // b, p.pad_w // b)
                       for b in sizes]
        fin = self.levels[-1]
        self.b_final = sizes[-1]
        self.gh, self.gw = fin.gh, fin.gw
        self.mv_ref = torch.empty_like(fin.mv)
        self.e_ref = torch.empty_like(fin.energy)
        self.replaced = torch.empty(fin.energy.shape, dtype=torch.int32, device=self.dev)
        coarse = sizes[0]
        self.ch, self.cw = p.pad_h // coarse, p.pad_w // coarse
        self.sp = N.select_params(self.gh, self.gw, coarse // self.b_final, self.ch, self.cw, config.aem_statistic,
                                  config.reference_policy, config.max_gop, config.aem_threshold)
        # AEM state zeroed at the start of every step: one byte buffer carved into
        # typed views (8-byte aligned) so the reset is one fill + the ref fill
        n_acc, n_tr = S * self.ch * self.cw, S * T
        n_i32 = 2 * S + S * T
        n_i32 += n_i32 % 2
        self._aem_zero = torch.zeros(8 * (n_acc + n_tr) + 4 * n_i32, dtype=torch.uint8, device=self.dev)
        z = self._aem_zero
        self.acc = z[:8 * n_acc].view(torch.float64).view(S, self.ch, self.cw)
        self.trigger = z[8 * n_acc:8 * (n_acc + n_tr)].view(torch.float64).view(S, T)
        ints = z[8 * (n_acc + n_tr):].view(torch.int32)
        self.fsk = ints[:S]
        self.last_key = ints[S:2 * S]
        self.kind = ints[2 * S:2 * S + S * T].view(S, T)
        self.ref = torch.full((S, T), -1, dtype=torch.int32, device=self.dev)
        self.workspace = torch.zeros(4, dtype=torch.int32, device=self.dev)  # label-chain grid barrier
        self.set_label_size(*(label_hw or (self.H, self.W)))
        self.graph = None

    # ------------------------------------------------------------------ buffers
    def set_label_size(self, h: int, w: int) -> None:
        B = self.b_final * self.scale
        if self.gw * B < w or self.gh * B < h:
            raise ValueError(f"motion field covers {self.gw * B}x{self.gh * B}, labels are {w}x{h}")
        self.Hl, self.Wl = int(h), int(w)
        self.labels = self.torch.zeros((self.S, self.T, h, w), dtype=self.torch.uint8, device=self.dev)
        self.key_labels = self.torch.zeros_like(self.labels)
        # CaBR weight-free fallback (ring vote) runs inside the label chain when refinement is on
        self.ring_vote = bool(self.cfg.refine_enabled)
        self.cabr = None
        self.graph = None

    def set_cabr(self, weights) -> None:
        """Refine flagged blocks with the CaBR-Net forward pass (cabr.py:306-345, weights given)
        instead of the ring vote: the label chain becomes bmc_cabr_chain."""
        from .cabr import packed_weights
        if not self.cfg.refine_enabled:
            raise ValueError("CaBR weights need refine_enabled")
        if (self.Hl, self.Wl) != (self.H, self.W):
            raise ValueError("frame and label map dimensions differ")
        torch, lib = self.torch, N.load()
        ws = lib.bmc_cabr_chain_workspace(self.S, self.T, self.gh, self.gw)
        self.cabr = dict(packed=packed_weights(weights, torch, self.dev), C=weights.num_classes,
                         scratch=torch.empty((self.S, self.Hl, self.Wl), dtype=torch.uint8, device=self.dev),
                         workspace=torch.empty((ws + 3) // 4, dtype=torch.int32, device=self.dev))
        self.graph = None

    def load_frames(self, frames, non_blocking: bool = False) -> None:
        """Copy (S, T, H, W) or (T, H, W) frames (numpy / CPU or CUDA tensor) into the raw slot."""
        src = frames
        if isinstance(src, np.ndarray):
            src = self.torch.from_numpy(np.ascontiguousarray(src))
        self.raw.view(-1, self.H, self.W).copy_(src.reshape(-1, self.H, self.W), non_blocking=non_blocking)

    # ------------------------------------------------------------------ stages
    def _level_slice(self, lo: int, hi: int):
        out = []
        for lv in self.levels:
            out.append(N.LevelOut(N.ptr(lv.mv[lo:hi]), N.ptr(lv.energy[lo:hi]), N.ptr(lv.matched[lo:hi]),
                                  N.ptr(lv.evals[lo:hi])))
        return (N.LevelOut * len(out))(*out)

    def _reset_state(self) -> None:
        N.memset_async(self._aem_zero, 0)  # acc, trigger, frames_since_key, last_key, kind
        N.memset_async(self.ref, 0xFF)  # int32 -1
        if self.cfg.reference_policy == "keyframe":
            self.ref_index.copy_(self.ref_index_init)

    def _decide(self, t0: int, t1: int, ref_next=None) -> None:
        cells = self.gh * self.gw
        S = self.S
        N.check(N.load().bmc_decide(
            N.ptr(self.e_ref) - 8 * S * cells, S * cells, cells, S, t0, t1, ctypes.byref(self.sp),
            N.ptr(self.acc), N.ptr(self.fsk), N.ptr(self.last_key), N.ptr(self.kind), N.ptr(self.ref),
            N.ptr(self.trigger), self.T, ref_next, self.T, N.stream_handle()))

    def _pack(self) -> None:
        N.check(N.load().bmc_pack_planes(N.ptr(self.raw), self.S * self.T, self.kind_code, ctypes.byref(self.params),
                                         N.ptr(self.planes), N.stream_handle()))

    def _estimate_all(self) -> None:
        arr = self._level_slice(0, self.n_pairs)
        N.check(N.load().bmc_estimate_motion(N.ptr(self.planes), self.S * self.T, ctypes.byref(self.params),
                                             self.n_pairs, N.ptr(self.cur_index), N.ptr(self.ref_index), arr,
                                             N.stream_handle()))

    def motion(self) -> None:
        """Pack + ME + refine + AEM decisions for every frame of every stream."""
        lib = N.load()
        p = self.params
        st = N.stream_handle()
        self._pack()
        self._reset_state()
        if self.T < 2:
            return
        if self.cfg.reference_policy == "previous":
            self._estimate_all()
            self._refine(0, self.n_pairs)
            self._decide(1, self.T)
            return
        S = self.S
        for t in range(1, self.T):
            lo, hi = (t - 1) * S, t * S
            arr = self._level_slice(lo, hi)
            N.check(lib.bmc_estimate_motion(N.ptr(self.planes), self.S * self.T, ctypes.byref(p), S, N.ptr(self.cur_index[lo:hi]),
                                            N.ptr(self.ref_index[lo:hi]), arr, st))
            self._refine(lo, hi)
            nxt = N.ptr(self.ref_index[hi:hi + S]) if t + 1 < self.T else None
            self._decide(t, t + 1, nxt)

    def launches_per_step(self) -> int:
        """Kernels of this library one step launches (pack, ME stages, refine, decide, label chain)."""
        fme = self.cfg.fme
        searched = 0
        for k, st in enumerate(fme.stages):
            if not (st.range == 0 and k > 0):  # range-0 stages after a searched stage are folded (no launch)
                searched += 1
        fpl = max(1, 65535 // (self.params.pad_h * (2 if self.bayer else 1)))  # frames per pack launch
        pack = -(-(self.S * self.T) // fpl)
        if self.cfg.reference_policy == "previous" or self.T < 2:
            motion = searched * len(fme.block_sizes) + (2 if self.T >= 2 else 0)
        else:
            motion = (self.T - 1) * (searched * len(fme.block_sizes) + 2)
        chain = 1 + 3 * self.T if self.cabr is not None else 1  # flag list + (predict, network, write-back) per frame
        return pack + motion + chain

    def _refine(self, lo: int, hi: int) -> None:
        fin = self.levels[-1]
        N.check(N.load().bmc_refine_mvs(
            N.ptr(fin.mv[lo:hi]), N.ptr(fin.energy[lo:hi]), hi - lo, self.gh, self.gw, self.b_final,
            int(self.cfg.deviation_threshold), N.ptr(self.planes), ctypes.byref(self.params),
            N.ptr(self.cur_index[lo:hi]), N.ptr(self.ref_index[lo:hi]), N.ptr(self.mv_ref[lo:hi]),
            N.ptr(self.e_ref[lo:hi]), N.ptr(self.replaced[lo:hi]), N.stream_handle()))

    def _chain(self, t0: int, t1: int) -> None:
        """Label chain of frames [t0, t1) of every stream (one cooperative launch); with
        refine_enabled the flagged blocks of predicted frames get CaBR's ring vote, or
        the network (set_cabr) frame by frame."""
        cells = self.gh * self.gw
        cells2 = cells * 2
        fs = self.Hl * self.Wl
        if self.cabr is not None:
            c = self.cabr
            N.check(N.load().bmc_cabr_chain(
                N.ptr(self.labels), fs, self.T * fs, N.ptr(self.key_labels), self.S, t0, t1, N.ptr(self.kind),
                N.ptr(self.ref), self.T, self.Hl, self.Wl, N.ptr(self.mv_ref) - 4 * self.S * cells2,
                self.S * cells2, cells2, self.gh, self.gw, self.b_final, self.scale,
                N.ptr(self.levels[-1].matched) - self.S * cells, N.ptr(self.raw),
                0 if self.raw.dtype == self.torch.uint8 else 1, self.H * self.W, self.T * self.H * self.W, c["C"],
                N.ptr(c["packed"]), N.ptr(c["scratch"]), N.ptr(c["workspace"]), N.stream_handle()))
            return
        ring = self.ring_vote
        matched = (N.ptr(self.levels[-1].matched) - self.S * cells) if ring else None
        N.check(N.load().bmc_predict_labels_clip(
            N.ptr(self.labels), fs, self.T * fs, N.ptr(self.key_labels), self.S, t0, t1, N.ptr(self.kind),
            N.ptr(self.ref), self.T, self.Hl, self.Wl, N.ptr(self.mv_ref) - 4 * self.S * cells2,
            self.S * cells2, cells2, self.gh, self.gw, self.b_final, self.scale, matched,
            None, N.ptr(self.workspace), N.stream_handle()))

    def predict(self) -> None:
        """Label chain (one cooperative launch): key frames copy key_labels, others gather from their reference."""
        self._chain(0, self.T)

    def step(self) -> None:
        self.motion()
        self.predict()

    # ------------------------------------------------------------------ graphs
    def capture(self) -> None:
        """Capture one full step as CUDA graphs.  With the "previous" policy the
        step is three graphs -- pack, motion estimation, and refine + AEM +
        label chain -- so a caller can bracket the ME graph with events
        (``replay(me_events=...)``) and time the dominant kernel inside a
        timed step; otherwise one graph."""
        torch = self.torch
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            self.step()  # warm-up: sets kernel attributes, builds tables
        torch.cuda.current_stream().wait_stream(side)
        if self.cfg.reference_policy == "previous" and self.T >= 2:
            graphs = []
            for part in (self._graph_pre, self._estimate_all, self._graph_post):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    part()
                graphs.append(g)
            self.graph = graphs
        else:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self.step()
            self.graph = [g]

    def _graph_pre(self) -> None:
        self._pack()
        self._reset_state()

    def _graph_post(self) -> None:
        self._refine(0, self.n_pairs)
        self._decide(1, self.T)
        self.predict()

    def replay(self, me_events=None) -> None:
        """Replay the captured step; ``me_events=(start, end)`` are recorded
        around the motion-estimation graph on the current stream."""
        if self.graph is None:
            self.capture()
        if len(self.graph) == 3 and me_events is not None:
            self.graph[0].replay()
            me_events[0].record()
            self.graph[1].replay()
            me_events[1].record()
            self.graph[2].replay()
            return
        for g in self.graph:
            g.replay()

    # ------------------------------------------------------------------ results
    def decisions_host(self):
        return self.kind.cpu().numpy(), self.ref.cpu().numpy(), self.trigger.cpu().numpy()

    def level_host(self, level: int):
        lv = self.levels[level]
        return (lv.mv[:self.n_pairs].cpu().numpy(), lv.energy[:self.n_pairs].cpu().numpy(),
                lv.matched[:self.n_pairs].cpu().numpy(), lv.evals[:self.n_pairs].cpu().numpy())

    def refined_host(self):
        return (self.mv_ref[:self.n_pairs].cpu().numpy(), self.e_ref[:self.n_pairs].cpu().numpy(),
                self.replaced[:self.n_pairs].cpu().numpy())

    def pair_index(self, s: int, t: int) -> int:
        return (t - 1) * self.S + s
