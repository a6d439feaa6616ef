"""Golden fixtures for the CaBR-Net path, made by running the REFERENCE (bayermc 0.1.0).

Run in the build container (where /root/reference is mounted):
    BAYERMC_THREADS=1 python tests/golden/make_golden_cabr.py
Writes tests/golden/cabr_*.npz:

* cabr_blocks.npz -- one Bayer frame + label map, seeded weights
  (random_weights(C, seed)), block origins for K = 16 / 32 / 64 including
  frame-border and partially-outside blocks: the reference's
  cabr_forward(extract_patch(...)) logits, extract_patch of one block, and
  refine_blocks outputs with and without weights.
* cabr_pipe_*.npz -- run_sequence(..., weights) over seeded clips whose
  predicted frames have flagged blocks (K = 16, 32, 64), plus per frame the
  smallest gap between the two best logits over every refined pixel, recorded
  from the reference's own forward passes (a label can only legitimately differ
  where that gap is within float32 rounding).

Inputs are regenerated from the seeds in the tests (synth is bit-identical to
the reference's generator) and their hashes stored.
"""

from __future__ import annotations

import hashlib
import os
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(HERE.parents[1]))
os.environ.setdefault("BAYERMC_THREADS", "1")

from bayermc import cabr, fme, frame_io, pipeline  # noqa: E402
from bayermc.config import PipelineConfig  # noqa: E402

from paper_2508_05990_b200 import synth  # noqa: E402


def digest(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


BLOCK_ORIGINS = {
    16: [(0, 0), (16, 32), (144, 112), (150, 120), (72, 40), (8, 100)],
    32: [(0, 0), (32, 64), (128, 96), (140, 110), (64, 32)],
    64: [(0, 0), (64, 64), (120, 90)],
}


def block_fixtures():
    w, h = 160, 128
    clip = synth.bayer_pan_clip(w, h, 2, (3, 1), seed=4)
    lab = synth.block_labels(w, h, 1, num_classes=7, seed=2)[0]
    fr = frame_io.Frame(w, h, clip[0], frame_io.FrameKind.BAYER_RGGB)
    wts = cabr.random_weights(lab.num_classes, seed=5)
    out = {"clip_hash": np.str_(digest(clip)), "num_classes": np.int64(lab.num_classes), "seed": np.int64(5)}
    for k, origins in BLOCK_ORIGINS.items():
        logits = np.stack([cabr.cabr_forward(cabr.extract_patch(fr, lab, o, k), wts) for o in origins])
        out[f"origins_{k}"] = np.array(origins, np.int32)
        out[f"logits_{k}"] = logits
        out[f"refined_{k}"] = cabr.refine_blocks(fr, lab, origins, k, wts).classes
        out[f"ringvote_{k}"] = cabr.refine_blocks(fr, lab, origins, k, None).classes
    p = cabr.extract_patch(fr, lab, (150, 120), 16)
    out["patch_image"], out["patch_context"] = p.image, p.context
    # uint16 frame (values divided by 65535) and a float frame in [0, 1]
    c16 = synth.bayer_pan_clip(w, h, 1, (0, 0), seed=6, dtype=np.uint16)
    out["clip16_hash"] = np.str_(digest(c16))
    f16 = frame_io.Frame(w, h, c16[0], frame_io.FrameKind.BAYER_RGGB)
    out["logits16_u16"] = np.stack([cabr.cabr_forward(cabr.extract_patch(f16, lab, o, 16), wts)
                                    for o in BLOCK_ORIGINS[16]])
    np.savez_compressed(HERE / "cabr_blocks.npz", **out)


class GapRecorder:
    """Wraps the reference's cabr_forward to record top-2 logit gaps of every refined block."""

    def __init__(self):
        self.min_gap = np.inf
        self.orig = cabr.cabr_forward

    def __call__(self, patch, weights):
        logits = self.orig(patch, weights)
        if logits.shape[0] > 1:
            s = np.sort(logits, axis=0)
            self.min_gap = min(self.min_gap, float((s[-1] - s[-2]).min()))
        return logits


def pipe_fixture(name, clip, labels, pcfg, seed):
    frames = [frame_io.Frame(clip.shape[2], clip.shape[1], c, frame_io.FrameKind.BAYER_RGGB) for c in clip]
    wts = cabr.random_weights(labels[0].num_classes, seed=seed)
    rec = GapRecorder()
    cabr.cabr_forward = rec
    try:
        res = pipeline.run_sequence(frames, {i: l for i, l in enumerate(labels)}, pcfg, weights=wts)
    finally:
        cabr.cabr_forward = rec.orig
    kinds = np.array([["key", "nonkey_prev_ref", "nonkey_key_ref"].index(d.kind.value) for d in res.decisions])
    refs = np.array([-1 if d.reference_index is None else d.reference_index for d in res.decisions])
    print(name, "keyframes", res.keyframes, "cabr flops", res.ledger["cabr"], "min gap", rec.min_gap)
    np.savez_compressed(HERE / f"cabr_pipe_{name}.npz", clip_hash=np.str_(digest(clip)),
                        out_labels=np.stack([l.classes for l in res.labels]), kinds=kinds, refs=refs,
                        ledger_cabr=np.int64(res.ledger["cabr"]), ledger_fme=np.int64(res.ledger["fme"]),
                        ledger_refine=np.int64(res.ledger["mv_refine"]), min_gap=np.float64(rec.min_gap),
                        seed=np.int64(seed), num_classes=np.int64(labels[0].num_classes))


def pipeline_fixtures():
    # K = 64: C5-style clip (standard preset, 64 -> 32 plane blocks), fixed GOP so frames are predicted
    w, h, t = 320, 256, 6
    clip = synth.bayer_pan_clip(w, h, t, (6, -4), seed=8, square=48, square_velocity=(7, 3))
    lab = synth.block_labels(w, h, t, num_classes=5, seed=1)
    pipe_fixture("k64", clip, lab, PipelineConfig(fme=fme.get_preset("standard"), max_gop=6,
                                                  aem_threshold=float("inf")), seed=7)
    # K = 32: 16-plane blocks, full +-8 then a +-1 refinement stage
    f1 = fme.FmeConfig(stages=(fme.SearchStage(8, 1), fme.SearchStage(0, 1), fme.SearchStage(1, 1)), block_sizes=(16,))
    c1 = synth.bayer_pan_clip(256, 192, 6, (3, 5), seed=31, square=64, square_velocity=(-5, 3))
    pipe_fixture("k32", c1, synth.block_labels(256, 192, 6, num_classes=6, seed=3),
                 PipelineConfig(fme=f1, max_gop=6, aem_threshold=float("inf")), seed=11)
    # K = 16: 16 -> 8 plane blocks
    f2 = fme.FmeConfig(stages=(fme.SearchStage(4, 2), fme.SearchStage(1, 1), fme.SearchStage(1, 1)),
                       block_sizes=(16, 8))
    c2 = synth.bayer_pan_clip(160, 128, 5, (2, -3), seed=12, square=40, square_velocity=(6, 2))
    pipe_fixture("k16", c2, synth.block_labels(160, 128, 5, num_classes=4, seed=9),
                 PipelineConfig(fme=f2, max_gop=5, aem_threshold=float("inf")), seed=14)


if __name__ == "__main__":
    block_fixtures()
    pipeline_fixtures()
