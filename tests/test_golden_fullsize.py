"""GPU parity at BASELINE.json's FULL sizes against the REFERENCE's own outputs.

The fixtures ``tests/golden/full_*.npz`` were produced by running bayermc 0.1.0
itself (``tests/golden/make_golden_fullsize.py``) on the bench's seeded clips:

* C2  1080p u8, b16, full +-16: every one of the 29 pairs, every block (mv, energy
  bits, matched, candidate_evals), the refined field of every pair, and
  ``run_sequence`` over the clip (default AEM 0.15; GOP-6 ring-vote variant);
* C2sq  C2 plus a textured square at an odd velocity (outliers, replacements);
* C3  4K u16, b8, stages (4,8)(2,4)(2,1) (the small-block kernel): pairs 1-3 and
  ``run_sequence`` over all 60 frames;
* C4  sample streams 0, 21, 63 (seed 1000+k, SURVEY velocities): pairs 1-3;
* C5  1080p standard preset, velocity sweep + square + scene cut: all 39 pairs at
  both levels and run_sequence in five variants (default, max_gop=5 & aem=inf,
  mean statistic, keyframe policy, ring vote).

Inputs are regenerated from the recipe and checked against the stored per-frame
SHA-256 before anything is compared.  Everything is bit-exact (float64 energies
and AEM triggers compared as int64 bit patterns).
"""

import hashlib

import numpy as np
import pytest

import golden_io as G

pytestmark = pytest.mark.gpu

CODES = {"key": 0, "nonkey_prev_ref": 1, "nonkey_key_ref": 2}


def bits(a):
    return np.asarray(a, dtype=np.float64).view(np.int64)


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).digest()


def _clip_for(name):
    from paper_2508_05990_b200 import synth
    if name == "c2":
        return synth.bayer_pan_clip(1920, 1080, 30, (4, -2), seed=5), synth.block_labels(1920, 1080, 30, seed=5)
    if name == "c2sq":
        return synth.bayer_pan_clip(1920, 1080, 4, (4, -2), seed=5, square=160, square_velocity=(7, -3)), None
    if name == "c3":
        return (synth.bayer_pan_clip(3840, 2160, 60, (6, -4), seed=11, dtype=np.uint16),
                synth.block_labels(3840, 2160, 60, seed=11))
    if name.startswith("c4s"):
        k = int(name[3:])
        v = (2 * ((k % 9) - 4), 2 * ((k // 9 % 7) - 3))
        return synth.bayer_pan_clip(1920, 1080, 4, v, seed=1000 + k), None
    if name == "c5":
        return synth.c5_clip(), synth.block_labels(1920, 1080, 40, seed=7)
    raise KeyError(name)


_CACHE = {}


def _load(name):
    if name not in _CACHE:
        d = G.load(f"full_{name}.npz")
        clip, labels = _clip_for(name)
        assert clip.shape == tuple(d["shape"]) and clip.dtype.name == str(d["dtype"])
        got = np.frombuffer(b"".join(_sha(c) for c in clip), np.uint8).reshape(-1, 32)
        np.testing.assert_array_equal(got, d["frame_sha"], err_msg="regenerated input differs from the fixture's")
        _CACHE.clear()  # keep one 4K clip resident at a time
        _CACHE[name] = (d, clip, labels)
    return _CACHE[name]


FIXTURES = ["c2", "c2sq", "c3", "c4s0", "c4s21", "c4s63", "c5"]


@pytest.mark.parametrize("name", FIXTURES)
def test_fullsize_every_block_matches_reference(cuda, name):
    """estimate_motion + refine_mvs(cur, ref, config) for the fixture's pairs, every block."""
    from paper_2508_05990_b200 import fme, mv_refine, synth
    d, clip, _ = _load(name)
    cfg = G.fme_config(d)
    frames = synth.frames_of(clip)
    pairs = [(int(t), int(t) - 1) for t in d["pairs"]]
    got = fme.estimate_motion_pairs(frames, pairs, cfg)
    nlev = int(d["levels"])
    for (t, r), fields in zip(pairs, got, strict=True):
        assert len(fields) == nlev
        for lv, f in enumerate(fields):
            k = f"P{t}L{lv}_"
            np.testing.assert_array_equal(f.mv, d[k + "mv"], err_msg=f"{name} pair {t} level {lv} mv")
            np.testing.assert_array_equal(bits(f.energy), bits(d[k + "energy"]),
                                          err_msg=f"{name} pair {t} level {lv} energy")
            np.testing.assert_array_equal(f.matched, d[k + "matched"], err_msg=f"{name} pair {t} level {lv} mask")
            assert f.candidate_evals == int(d[k + "evals"]), (name, t, lv)
        ref_f = mv_refine.refine_mvs(fields[-1], 4, cur=frames[t], ref=frames[r], config=cfg)
        np.testing.assert_array_equal(ref_f.mv, d[f"P{t}R_mv"], err_msg=f"{name} pair {t} refined mv")
        np.testing.assert_array_equal(bits(ref_f.energy), bits(d[f"P{t}R_energy"]),
                                      err_msg=f"{name} pair {t} refined energy")


VARIANTS = [("c2", "default"), ("c2", "ringvote"), ("c3", "default"), ("c5", "default"), ("c5", "gop5"),
            ("c5", "mean"), ("c5", "keyframe"), ("c5", "ringvote")]


def _pipeline_config(d, v):
    from paper_2508_05990_b200.config import PipelineConfig
    gop = int(d[f"{v}_max_gop"])
    return PipelineConfig(fme=G.fme_config(d), refine_enabled=bool(d[f"{v}_refine"]),
                          aem_threshold=float(d[f"{v}_aem"]), max_gop=gop or None,
                          aem_statistic=str(d[f"{v}_statistic"]), reference_policy=str(d[f"{v}_policy"]))


@pytest.mark.parametrize("name,variant", VARIANTS)
def test_fullsize_run_sequence_matches_reference(cuda, name, variant):
    """run_sequence over the whole clip: decisions, trigger bits, every label map, ledger."""
    from paper_2508_05990_b200 import pipeline, synth
    from paper_2508_05990_b200.frame_io import LabelMap
    d, clip, labels = _load(name)
    pcfg = _pipeline_config(d, variant)
    keys = {i: LabelMap(l.width, l.height, l.classes, l.num_classes) for i, l in enumerate(labels)}
    res = pipeline.run_sequence(synth.frames_of(clip), keys, pcfg)
    np.testing.assert_array_equal([CODES[x.kind.value] for x in res.decisions], d[f"{variant}_kinds"])
    np.testing.assert_array_equal([-1 if x.reference_index is None else x.reference_index for x in res.decisions],
                                  d[f"{variant}_refs"])
    np.testing.assert_array_equal(bits([x.trigger_statistic for x in res.decisions]), bits(d[f"{variant}_trig"]))
    got_sha = np.frombuffer(b"".join(_sha(l.classes) for l in res.labels), np.uint8).reshape(-1, 32)
    bad = [i for i in range(len(res.labels)) if not np.array_equal(got_sha[i], d[f"{variant}_label_sha"][i])]
    assert not bad, f"{name}/{variant}: label maps differ at frames {bad}"
    for k in ("fme", "mv_refine", "prediction", "backbone", "cabr"):
        assert res.ledger[k] == int(d[f"{variant}_ledger_{k}"]), (name, variant, k)


def test_fullsize_fixtures_exercise_prediction():
    """The variants above must include real compensation (non-key frames), not only keys."""
    predicted = 0
    for name, v in VARIANTS:
        d = G.load(f"full_{name}.npz")
        predicted += int((d[f"{v}_kinds"] != 0).sum())
    assert predicted > 50


def test_fullsize_clip_engine_c2_matches_reference(cuda):
    """The bench's own engine path (ClipEngine graphs, the measured code) on the C2 clip."""
    from paper_2508_05990_b200.engine import ClipEngine
    d, clip, labels = _load("c2")
    pcfg = _pipeline_config(d, "default")
    eng = ClipEngine(pcfg, 1080, 1920, 30)
    eng.load_frames(clip)
    for t in range(30):
        eng.key_labels[0, t].copy_(cuda.from_numpy(labels[t].classes))
    eng.capture()
    eng.replay()
    cuda.cuda.synchronize()
    mv0, e0, m0, ev0 = eng.level_host(0)
    mvr, er, _ = eng.refined_host()
    for t in range(1, 30):
        p = eng.pair_index(0, t)
        np.testing.assert_array_equal(mv0[p], d[f"P{t}L0_mv"])
        np.testing.assert_array_equal(bits(e0[p]), bits(d[f"P{t}L0_energy"]))
        np.testing.assert_array_equal(m0[p].astype(bool), d[f"P{t}L0_matched"])
        np.testing.assert_array_equal(mvr[p], d[f"P{t}R_mv"])
        np.testing.assert_array_equal(bits(er[p]), bits(d[f"P{t}R_energy"]))
    kinds, refs, trig = (a[0] for a in eng.decisions_host())
    np.testing.assert_array_equal(kinds, d["default_kinds"])
    np.testing.assert_array_equal(bits(trig), bits(d["default_trig"]))
    out = eng.labels[0].cpu().numpy()
    for t in range(30):
        assert _sha(out[t]) == bytes(d["default_label_sha"][t]), t
