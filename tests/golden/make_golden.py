"""Generate golden fixtures by running the REFERENCE package (bayermc 0.1.0).

Run in the build container (where /root/reference is mounted):
    BAYERMC_THREADS=1 python tests/golden/make_golden.py
Writes tests/golden/*.npz.  Inputs are regenerated from seeds where possible
and stored when small, so GPU tests on a box without the reference can compare
the CUDA path directly against the reference's own outputs.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))
sys.path.insert(0, str(HERE.parents[1]))
os.environ.setdefault("BAYERMC_THREADS", "1")

from bayermc import fme, frame_io, frame_select, mv_refine, pipeline, propagate  # noqa: E402
from bayermc.config import PipelineConfig  # noqa: E402

from paper_2508_05990_b200 import synth  # noqa: E402  (seeded Bayer clip recipe; value_noise == reference's)


def fields_dict(prefix, fields):
    out = {}
    for lv, f in enumerate(fields):
        out[f"{prefix}L{lv}_mv"] = np.asarray(f.mv)
        out[f"{prefix}L{lv}_energy"] = np.asarray(f.energy)
        out[f"{prefix}L{lv}_matched"] = np.asarray(f.matched)
        out[f"{prefix}L{lv}_evals"] = np.int64(f.candidate_evals)
        out[f"{prefix}L{lv}_block"] = np.int64(f.block_size)
    out[f"{prefix}levels"] = np.int64(len(fields))
    return out


def cfg_arrays(c):
    return {"stages": np.array([[s.range, s.step] for s in c.stages], np.int64), "lam": np.float64(c.lam),
            "block_sizes": np.array(c.block_sizes, np.int64), "split": np.float64(c.split_threshold),
            "tol": np.float64(c.sparsity_tolerance), "refine_thr": np.float64(c.refine_block_threshold)}


ME_CASES = [
    # name, (h, w), hi, dtype, bayer, config
    ("std_bayer_u8", (128, 128), 256, np.uint8, True, fme.get_preset("standard")),
    ("full8_b16_bayer", (96, 160), 256, np.uint8, True,
     fme.FmeConfig(stages=(fme.SearchStage(8, 1), fme.SearchStage(0, 1), fme.SearchStage(0, 1)), block_sizes=(16,))),
    ("full8_b16_luma_lowc", (70, 54), 10, np.uint8, False,
     fme.FmeConfig(stages=(fme.SearchStage(8, 1), fme.SearchStage(0, 1), fme.SearchStage(0, 1)), block_sizes=(16,))),
    ("chain_b16_8_u16", (128, 128), 65536, np.uint16, True,
     fme.FmeConfig(stages=(fme.SearchStage(4, 1), fme.SearchStage(0, 1), fme.SearchStage(1, 1)),
                   block_sizes=(16, 8), lam=0.3)),
    ("steps_b8_u16", (80, 80), 256, np.uint16, True,
     fme.FmeConfig(stages=(fme.SearchStage(2, 2), fme.SearchStage(1, 3), fme.SearchStage(2, 1)), block_sizes=(8,),
                   lam=0.5)),
    ("lam1_b8", (48, 40), 5, np.uint8, True,
     fme.FmeConfig(stages=(fme.SearchStage(2, 1), fme.SearchStage(1, 1), fme.SearchStage(1, 1)), block_sizes=(8,),
                   lam=1.0)),
    ("mode4_bayer", (256, 192), 256, np.uint8, True, fme.get_preset("mode4")),
]


def me_fixtures():
    rng = np.random.default_rng(2024)
    out = {}
    for name, (h, w), hi, dt, bayer, cfg in ME_CASES:
        kind = frame_io.FrameKind.BAYER_RGGB if bayer else frame_io.FrameKind.LUMA
        a = rng.integers(0, hi, (h, w)).astype(dt)
        b = rng.integers(0, hi, (h, w)).astype(dt)
        fields = fme.estimate_motion(frame_io.Frame(w, h, a, kind), frame_io.Frame(w, h, b, kind), cfg)
        d = {"cur": a, "ref": b, "bayer": np.bool_(bayer), **cfg_arrays(cfg), **fields_dict("", fields)}
        np.savez_compressed(HERE / f"me_{name}.npz", **d)
        out[name] = d
    # low-contrast tie fixture (SURVEY §8c fixture 4)
    tcfg = fme.FmeConfig(stages=(fme.SearchStage(2, 1), fme.SearchStage(0, 1), fme.SearchStage(0, 1)), block_sizes=(8,))
    trng = np.random.default_rng(7)
    a = trng.integers(0, 10, (64, 64)).astype(np.uint8)
    b = trng.integers(0, 10, (64, 64)).astype(np.uint8)
    fields = fme.estimate_motion(frame_io.Frame(64, 64, a), frame_io.Frame(64, 64, b), tcfg)
    np.savez_compressed(HERE / "me_tie_lowcontrast.npz", cur=a, ref=b, bayer=np.bool_(False), **cfg_arrays(tcfg),
                        **fields_dict("", fields))


def pipeline_fixture(name, clip, labels, pcfg, store_inputs=True, inputs_from=None):
    frames = [frame_io.Frame(clip.shape[2], clip.shape[1], c, frame_io.FrameKind.BAYER_RGGB) for c in clip]
    res = pipeline.run_sequence(frames, {i: l for i, l in enumerate(labels)}, pcfg)
    kinds = np.array([["key", "nonkey_prev_ref", "nonkey_key_ref"].index(d.kind.value) for d in res.decisions])
    refs = np.array([-1 if d.reference_index is None else d.reference_index for d in res.decisions])
    trig = np.array([d.trigger_statistic for d in res.decisions])
    inputs = {"clip": clip, "key_labels": np.stack([l.classes for l in labels])} if store_inputs \
        else {"inputs_from": np.str_(inputs_from)}
    np.savez_compressed(HERE / f"pipe_{name}.npz", **inputs,
                        out_labels=np.stack([l.classes for l in res.labels]), kinds=kinds, refs=refs, trig=trig,
                        aem=np.float64(pcfg.aem_threshold), max_gop=np.int64(pcfg.max_gop or 0),
                        has_max_gop=np.bool_(pcfg.max_gop is not None), statistic=np.str_(pcfg.aem_statistic),
                        policy=np.str_(pcfg.reference_policy), refine=np.bool_(pcfg.refine_enabled),
                        ledger_fme=np.int64(res.ledger["fme"]),
                        ledger_refine=np.int64(res.ledger["mv_refine"]), **cfg_arrays(pcfg.fme))


def pipeline_fixtures():
    # C1: 256x256 RGGB uint8, 8 frames, v=(2,2), seed 3, b16 full +-8
    c1 = synth.bayer_pan_clip(256, 256, 8, (2, 2), seed=3)
    lab = synth.block_labels(256, 256, 8)
    f1 = fme.FmeConfig(stages=(fme.SearchStage(8, 1), fme.SearchStage(0, 1), fme.SearchStage(0, 1)), block_sizes=(16,))
    pipeline_fixture("c1", c1, lab, PipelineConfig(fme=f1, refine_enabled=False))
    # C5-style decisions: standard preset, moving square, scene cut, variants (reduced size)
    w, h, t = 320, 256, 10
    clip = synth.bayer_pan_clip(w, h, t, (6, -4), seed=8, square=48, square_velocity=(7, 3))
    clip[7:] = synth.bayer_pan_clip(w, h, t - 7, (2, 2), seed=99)
    lab = synth.block_labels(w, h, t)
    std = fme.get_preset("standard")
    pipeline_fixture("c5s_default", clip, lab, PipelineConfig(fme=std, refine_enabled=False))
    kw = dict(store_inputs=False, inputs_from="pipe_c5s_default.npz")
    pipeline_fixture("c5s_gop5", clip, lab, PipelineConfig(fme=std, refine_enabled=False, max_gop=5,
                                                           aem_threshold=float("inf")), **kw)
    pipeline_fixture("c5s_mean", clip, lab, PipelineConfig(fme=std, refine_enabled=False, aem_statistic="mean",
                                                           aem_threshold=0.05), **kw)
    pipeline_fixture("c5s_keyframe", clip, lab, PipelineConfig(fme=std, refine_enabled=False,
                                                               reference_policy="keyframe"), **kw)


def ringvote_fixtures():
    # refine_enabled=True without weights: CaBR's ring-vote fallback re-labels the flagged blocks of every
    # predicted frame and the refined labels feed the next frame's prediction (pipeline.py:123-135)
    w, h, t = 320, 256, 10
    clip = synth.bayer_pan_clip(w, h, t, (6, -4), seed=8, square=48, square_velocity=(7, 3))
    clip[7:] = synth.bayer_pan_clip(w, h, t - 7, (2, 2), seed=99)
    lab = synth.block_labels(w, h, t)
    std = fme.get_preset("standard")
    kw = dict(store_inputs=False, inputs_from="pipe_c5s_default.npz")
    pipeline_fixture("c5s_ringvote", clip, lab, PipelineConfig(fme=std), **kw)
    pipeline_fixture("c5s_ringvote_gop4", clip, lab, PipelineConfig(fme=std, max_gop=4, aem_threshold=float("inf")),
                     **kw)
    f1 = fme.FmeConfig(stages=(fme.SearchStage(8, 1), fme.SearchStage(0, 1), fme.SearchStage(1, 1)), block_sizes=(16,))
    c1 = synth.bayer_pan_clip(256, 192, 6, (3, 5), seed=31, square=64, square_velocity=(-5, 3))
    pipeline_fixture("ringvote_b16_odd", c1, synth.block_labels(256, 192, 6, seed=3),
                     PipelineConfig(fme=f1, max_gop=6, aem_threshold=float("inf")))


def kat_fixtures():
    out = {}
    # SPEC.md:130 block_energy single-pixel example
    a = np.zeros((64, 64))
    b = a.copy()
    b[3, 5] = 0.2
    out["kat_block_energy"] = np.float64(fme.block_energy(a, b, 0.1, 8 / 255))
    # SPEC.md:71 pack_bayer 4x4 example
    f = frame_io.Frame(4, 4, np.arange(16, dtype=np.uint8).reshape(4, 4), frame_io.FrameKind.BAYER_RGGB)
    out["kat_pack_bayer"] = np.stack([np.asarray(p) for p in frame_io.pack_bayer(f).planes])
    # SPEC.md:200 refine outlier example
    mv = np.zeros((3, 3, 2), np.int64)
    mv[..., 0] = 2
    mv[1, 1] = (30, -12)
    fld = fme.MotionField(16, 3, 3, mv, np.zeros((3, 3)), np.ones((3, 3), bool))
    out["kat_refine_in"] = mv
    out["kat_refine_out"] = np.asarray(mv_refine.refine_mvs(fld, 4).mv)
    # SPEC.md:279 decide example: 0.4/frame, threshold 1.0
    _, st = frame_select.open_gop(0, 2, 2, 16)
    kinds = []
    for i in range(1, 4):
        e = np.full((2, 2), 0.4)
        fl = fme.MotionField(16, 2, 2, np.zeros((2, 2, 2), np.int64), e, np.ones((2, 2), bool))
        d, st = frame_select.decide(st, fl, i, aem_threshold=1.0)
        kinds.append(d.kind.value)
    out["kat_decide_kinds"] = np.array(kinds)
    # propagate: random field + labels
    rng = np.random.default_rng(3)
    mvp = rng.integers(-20, 21, (4, 4, 2)).astype(np.int64)
    fl = fme.MotionField(16, 4, 4, mvp, np.zeros((4, 4)), np.ones((4, 4), bool))
    cls = rng.integers(0, 7, (100, 90)).astype(np.uint8)
    out["prop_mv"] = mvp
    out["prop_in"] = cls
    out["prop_out"] = np.asarray(propagate.predict_labels(frame_io.LabelMap(90, 100, cls, 7), fl, 2).classes)
    # count_fme_flops KATs
    out["kat_flops_one"] = np.int64(fme.flops_per_candidate(64))
    out["kat_flops_std"] = np.int64(fme.count_fme_flops((2048, 1024), fme.get_preset("standard"), 512 * 131))
    np.savez_compressed(HERE / "kats.npz", **out)


def decide_fixture():
    rng = np.random.default_rng(17)
    seqs = {}
    for statistic in ("max", "mean"):
        for max_gop in (None, 3):
            for policy in ("previous", "keyframe"):
                ch, cw, f = 9, 15, 2
                _, st = frame_select.open_gop(0, cw, ch, 32)
                last_key = 0
                es, kinds, refs, trigs = [], [], [], []
                for i in range(1, 9):
                    e = rng.random((ch * f, cw * f)) * 0.06
                    fl = fme.MotionField(16, cw * f, ch * f, np.zeros((ch * f, cw * f, 2), np.int64), e,
                                         np.ones_like(e, bool))
                    d, st = frame_select.decide(st, fl, i, 0.15, max_gop, statistic, policy, last_key)
                    es.append(e)
                    kinds.append(d.kind.value)
                    refs.append(-1 if d.reference_index is None else d.reference_index)
                    trigs.append(d.trigger_statistic)
                    if d.kind.value == "key":
                        last_key = i
                key = f"{statistic}_{max_gop}_{policy}"
                seqs[key + "_e"] = np.stack(es)
                seqs[key + "_kinds"] = np.array(kinds)
                seqs[key + "_refs"] = np.array(refs)
                seqs[key + "_trig"] = np.array(trigs)
    np.savez_compressed(HERE / "decide_sequences.npz", **seqs)


if __name__ == "__main__":
    only = sys.argv[1:]  # e.g. "ringvote": regenerate one group only
    if not only or "me" in only:
        me_fixtures()
    if not only or "pipeline" in only:
        pipeline_fixtures()
    if not only or "ringvote" in only:
        ringvote_fixtures()
    if not only or "kat" in only:
        kat_fixtures()
    if not only or "decide" in only:
        decide_fixture()
    np.savez_compressed(HERE / "meta.npz", numpy_version=np.str_(np.__version__))
    print("wrote", sorted(p.name for p in HERE.glob("*.npz")))
