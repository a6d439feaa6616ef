"""GPU parity: the sm_100a path through the C ABI vs the CPU oracle.

Integer outputs (MVs, masks, candidate counts, decisions, labels) must be
bit-exact; float64 energies and AEM triggers must be bit-exact too (the
north star's 1e-5 relative budget applies only to float features, which are
copies and therefore also exact).  Sizes are chosen so the oracle finishes in
seconds.
"""

import numpy as np
import pytest

from oracle import bayermc_oracle as O

pytestmark = pytest.mark.gpu


def ocfg(c):
    return O.cfg_dict(stages=[(s.range, s.step) for s in c.stages], lam=c.lam, block_sizes=c.block_sizes,
                      split_threshold=c.split_threshold, sparsity_tolerance=c.sparsity_tolerance,
                      refine_block_threshold=c.refine_block_threshold)


def assert_levels_equal(gpu_fields, oracle_fields):
    assert len(gpu_fields) == len(oracle_fields)
    for g, o in zip(gpu_fields, oracle_fields):
        assert g.block_size == o.block_size
        np.testing.assert_array_equal(g.mv, o.mv)
        np.testing.assert_array_equal(g.matched, o.matched)
        assert g.candidate_evals == o.candidate_evals
        # bit-exact float64
        np.testing.assert_array_equal(g.energy.view(np.int64), o.energy.view(np.int64))


def _frames(rng, h, w, hi, dtype, bayer):
    from paper_2508_05990_b200.frame_io import Frame, FrameKind
    kind = FrameKind.BAYER_RGGB if bayer else FrameKind.LUMA
    a = rng.integers(0, hi, (h, w)).astype(dtype)
    b = rng.integers(0, hi, (h, w)).astype(dtype)
    return Frame(w, h, a, kind), Frame(w, h, b, kind)


def _cfgs():
    from paper_2508_05990_b200.fme import FmeConfig, SearchStage, get_preset
    return {
        "standard": get_preset("standard"),
        "full8_b16": FmeConfig(stages=(SearchStage(8, 1), SearchStage(0, 1), SearchStage(0, 1)), block_sizes=(16,)),
        "chain_b16_8": FmeConfig(stages=(SearchStage(4, 1), SearchStage(0, 1), SearchStage(1, 1)),
                                 block_sizes=(16, 8), lam=0.3),
        "steps_b8": FmeConfig(stages=(SearchStage(2, 2), SearchStage(1, 3), SearchStage(2, 1)), block_sizes=(8,),
                              lam=0.5),
        "lam0": FmeConfig(stages=(SearchStage(3, 1), SearchStage(1, 2), SearchStage(1, 1)), block_sizes=(16,),
                          lam=0.0),
        "lam1": FmeConfig(stages=(SearchStage(2, 1), SearchStage(1, 1), SearchStage(1, 1)), block_sizes=(8,),
                          lam=1.0),
        "mode4": get_preset("mode4"),
        "mode5": get_preset("mode5"),
    }


CASES = [
    # (h, w, hi, dtype, bayer, cfg)
    (128, 128, 256, np.uint8, True, "standard"),
    (96, 160, 256, np.uint8, True, "full8_b16"),
    (70, 54, 10, np.uint8, False, "full8_b16"),
    (64, 96, 3, np.uint8, True, "chain_b16_8"),
    (80, 80, 256, np.uint16, True, "steps_b8"),
    (64, 64, 40, np.uint8, False, "lam0"),
    (48, 40, 5, np.uint8, True, "lam1"),
    (128, 128, 65536, np.uint16, True, "chain_b16_8"),
    (160, 144, 2000, np.uint16, False, "full8_b16"),
    (256, 192, 256, np.uint8, True, "mode4"),
    (192, 256, 256, np.uint8, True, "mode5"),
]


@pytest.mark.parametrize("case", range(len(CASES)))
def test_estimate_motion_random(cuda, case):
    from paper_2508_05990_b200 import fme
    h, w, hi, dt, bayer, cname = CASES[case]
    rng = np.random.default_rng(100 + case)
    cur, ref = _frames(rng, h, w, hi, dt, bayer)
    cfg = _cfgs()[cname]
    got = fme.estimate_motion(cur, ref, cfg)
    want = O.estimate_motion(O.search_planes(cur.data, bayer), O.search_planes(ref.data, bayer), ocfg(cfg))
    assert_levels_equal(got, want)


def test_low_contrast_tie_fixture(cuda):
    """SURVEY §8c fixture (4): integer (S, C) ties whose float64 energies differ."""
    from paper_2508_05990_b200 import fme
    from paper_2508_05990_b200.fme import FmeConfig, SearchStage
    cfg = FmeConfig(stages=(SearchStage(2, 1), SearchStage(0, 1), SearchStage(0, 1)), block_sizes=(8,))
    rng = np.random.default_rng(7)
    for trial in range(12):
        cur, ref = _frames(rng, 64, 64, 10, np.uint8, trial % 2 == 0)
        got = fme.estimate_motion(cur, ref, cfg)
        want = O.estimate_motion(O.search_planes(cur.data, cur.kind.is_bayer),
                                 O.search_planes(ref.data, ref.kind.is_bayer), ocfg(cfg))
        assert_levels_equal(got, want)


def test_sparsity_boundary_pairs(cuda):
    """The 16 uint8 pairs with |a-b| = 8 that count as sparse."""
    from paper_2508_05990_b200 import fme
    from paper_2508_05990_b200.fme import FmeConfig, SearchStage
    from paper_2508_05990_b200.frame_io import Frame, FrameKind
    special = [25, 27, 29, 31, 58, 62, 124, 125, 33, 35, 37, 39, 66, 70, 132, 133]
    rng = np.random.default_rng(11)
    a = rng.choice(special, size=(64, 64)).astype(np.uint8)
    b = np.where(rng.random((64, 64)) < 0.5, a + 8, a - 8).clip(0, 255).astype(np.uint8)
    cfg = FmeConfig(stages=(SearchStage(1, 1), SearchStage(0, 1), SearchStage(0, 1)), block_sizes=(8,))
    for kind in (FrameKind.LUMA, FrameKind.BAYER_RGGB):
        cur, ref = Frame(64, 64, a, kind), Frame(64, 64, b, kind)
        got = fme.estimate_motion(cur, ref, cfg)
        want = O.estimate_motion(O.search_planes(a, kind.is_bayer), O.search_planes(b, kind.is_bayer), ocfg(cfg))
        assert_levels_equal(got, want)


def test_uint16_equals_uint8_times_257(cuda):
    from paper_2508_05990_b200 import fme, synth
    clip = synth.bayer_pan_clip(128, 96, 2, (3, 5), seed=4)
    f8 = synth.frames_of(clip)
    f16 = synth.frames_of(clip.astype(np.uint16) * 257)
    cfg = _cfgs()["chain_b16_8"]
    a = fme.estimate_motion(f8[1], f8[0], cfg)
    b = fme.estimate_motion(f16[1], f16[0], cfg)
    assert_levels_equal(a, b)


def test_identical_frames_zero_motion(cuda):
    from paper_2508_05990_b200 import fme, synth
    clip = synth.bayer_pan_clip(256, 128, 1, (0, 0), seed=1)
    f = synth.frames_of(clip)[0]
    out = fme.estimate_motion(f, f)
    assert all((lv.mv == 0).all() and (lv.energy == 0).all() for lv in out)
    assert out[0].matched.all()


def test_global_shift_recovery(cuda):
    """every even full-res shift in [-16,16] (plane [-8,8]) is recovered."""
    from paper_2508_05990_b200 import fme, synth
    from paper_2508_05990_b200.fme import FmeConfig, SearchStage
    cfg = FmeConfig(stages=(SearchStage(8, 1), SearchStage(0, 1), SearchStage(0, 1)), block_sizes=(16,))
    for vx, vy in [(-16, 0), (16, -16), (6, 10), (0, 0), (-8, 14)]:
        clip = synth.bayer_pan_clip(256, 256, 2, (vx, vy), seed=3)
        fr = synth.frames_of(clip)
        out = fme.estimate_motion(fr[1], fr[0], cfg)[0]
        inner = out.mv[1:-1, 1:-1]
        assert (inner[..., 0] == vx // 2).all() and (inner[..., 1] == vy // 2).all()


def test_search_stage_and_full_search(cuda):
    from paper_2508_05990_b200 import fme
    from paper_2508_05990_b200.fme import FmeConfig
    rng = np.random.default_rng(5)
    cfg = FmeConfig()
    for trial in range(6):
        bayer = trial % 2 == 0
        cur, ref = _frames(rng, 96, 80, 256 if trial < 3 else 6, np.uint8, bayer)
        pc, pr = O.search_planes(cur.data, bayer), O.search_planes(ref.data, bayer)
        h, w = pc.shape[1:]
        b = 8 if trial % 3 else 16
        ox, oy = int(rng.integers(0, w - b)), int(rng.integers(0, h - b))
        rng_, step = int(rng.integers(0, 5)), int(rng.integers(1, 4))
        center = (int(rng.integers(-3, 4)), int(rng.integers(-3, 4)))
        curb = np.ascontiguousarray(pc[:, oy:oy + b, ox:ox + b])
        want = O.stage_candidates(pr, curb, (ox, oy), b, center, rng_, step, cfg.lam, cfg.sparsity_tolerance)
        if want is None:
            with pytest.raises(ValueError):
                fme.search_stage(cur, ref, (ox, oy), b, center, rng_, step, cfg)
            continue
        mv, e = fme.search_stage(cur, ref, (ox, oy), b, center, rng_, step, cfg)
        assert mv == want[0] and e == want[1]
        mv2, e2 = fme.full_search(cur, ref, (ox, oy), b, 3, cfg)
        w2 = O.stage_candidates(pr, curb, (ox, oy), b, (0, 0), 3, 1, cfg.lam, cfg.sparsity_tolerance)
        assert mv2 == w2[0] and e2 == w2[1]


def test_block_energy(cuda):
    from paper_2508_05990_b200 import fme
    rng = np.random.default_rng(9)
    for shape in [(64, 64), (4, 16, 16), (3, 7, 5), (1, 1), (4, 100, 30)]:
        a, b = rng.random(shape), rng.random(shape)
        assert fme.block_energy(a, b, 0.1) == O.block_energy(a, b, 0.1)
    a = np.zeros((64, 64))
    b = a.copy()
    b[3, 5] = 0.2
    assert fme.block_energy(a, b, 0.1, 8 / 255) == O.block_energy(a, b, 0.1, 8 / 255)  # SPEC.md:130 KAT


def test_refine_mvs(cuda):
    from paper_2508_05990_b200 import fme, mv_refine
    rng = np.random.default_rng(21)
    cfg = _cfgs()["chain_b16_8"]
    for trial in range(4):
        cur, ref = _frames(rng, 128, 128, 256 if trial % 2 else 12, np.uint8, True)
        fields = fme.estimate_motion(cur, ref, cfg)
        fin = fields[-1]
        mv = fin.mv.copy()
        mv[rng.integers(0, fin.grid_h, 5), rng.integers(0, fin.grid_w, 5)] = rng.integers(-9, 10, (5, 2))
        noisy = fme.MotionField(fin.block_size, fin.grid_w, fin.grid_h, mv, fin.energy, fin.matched, fin.level,
                                fin.candidate_evals)
        got = mv_refine.refine_mvs(noisy, 2, cur=cur, ref=ref, config=cfg)
        of = O.OracleField(fin.block_size, mv.copy(), fin.energy.copy(), fin.matched.copy(), fin.level,
                           fin.candidate_evals)
        want = O.refine_mvs(of, 2, O.search_planes(cur.data, True), O.search_planes(ref.data, True), ocfg(cfg))
        np.testing.assert_array_equal(got.mv, want.mv)
        np.testing.assert_array_equal(got.energy.view(np.int64), want.energy.view(np.int64))
        np.testing.assert_array_equal(got.matched, fin.matched)
        nore = mv_refine.refine_mvs(noisy, 2)  # no cur/ref: energies kept
        np.testing.assert_array_equal(nore.energy, fin.energy)


def test_refine_spec_examples(cuda):
    from paper_2508_05990_b200 import fme, mv_refine
    mv = np.zeros((3, 3, 2), np.int64)
    mv[..., 0] = 2
    mv[1, 1] = (30, -12)
    f = fme.MotionField(16, 3, 3, mv, np.zeros((3, 3)), np.ones((3, 3), bool))
    out = mv_refine.refine_mvs(f, 4)
    assert (out.mv[..., 0] == 2).all() and (out.mv[..., 1] == 0).all()


def test_predict_labels_and_features(cuda):
    from paper_2508_05990_b200 import fme, propagate
    from paper_2508_05990_b200.frame_io import LabelMap
    rng = np.random.default_rng(3)
    for (h, w, b, scale) in [(100, 90, 8, 2), (64, 64, 16, 1), (33, 47, 8, 1), (540, 960, 16, 2)]:
        bs = b * scale
        gh, gw = -(-h // bs), -(-w // bs)
        mv = rng.integers(-20, 21, (gh, gw, 2)).astype(np.int64)
        field = fme.MotionField(b, gw, gh, mv, np.zeros((gh, gw)), np.ones((gh, gw), bool))
        cls = rng.integers(0, 7, (h, w)).astype(np.uint8)
        got = propagate.predict_labels(LabelMap(w, h, cls, 7), field, scale)
        want = O.predict_labels(cls, O.OracleField(b, mv, field.energy, field.matched, 0, 0), scale)
        np.testing.assert_array_equal(got.classes, want)
        feats = rng.random((3, h, w)).astype(np.float32)
        gf = propagate.predict_features(feats, [field], scale)
        wf = np.stack([feats[c][np.clip(np.arange(h)[:, None] + mv[np.arange(h)[:, None] // bs,
                                                                      np.arange(w)[None, :] // bs, 1] * scale, 0, h - 1),
                                np.clip(np.arange(w)[None, :] + mv[np.arange(h)[:, None] // bs,
                                                                   np.arange(w)[None, :] // bs, 0] * scale, 0, w - 1)]
                       for c in range(3)])
        np.testing.assert_array_equal(gf, wf)


def test_decide_sequences(cuda):
    from paper_2508_05990_b200 import fme, frame_select as fs
    rng = np.random.default_rng(17)
    for statistic in ("max", "mean"):
        for max_gop in (None, 3):
            for policy in ("previous", "keyframe"):
                for (ch, cw, f) in [(3, 5, 2), (9, 15, 1), (34, 60, 1)]:
                    state_g = fs.AemState.fresh(cw, ch, 32)
                    acc, fsk, last_key = np.zeros((ch, cw)), 0, 0
                    for i in range(1, 9):
                        e = rng.random((ch * f, cw * f)) * 0.06
                        field = fme.MotionField(32 // f, cw * f, ch * f, np.zeros((ch * f, cw * f, 2), np.int64), e,
                                                np.ones_like(e, bool))
                        d, state_g = fs.decide(state_g, field, i, 0.15, max_gop, statistic, policy, last_key)
                        kind, ref, trig, acc, fsk = O.decide(acc, fsk, 32, e, 32 // f, i, 0.15, max_gop, statistic,
                                                             policy, last_key)
                        assert d.kind.value == kind and d.reference_index == ref
                        assert d.trigger_statistic == trig
                        np.testing.assert_array_equal(state_g.accumulated, acc)
                        assert state_g.frames_since_key == fsk
                        if kind == "key":
                            last_key = i


def test_decide_spec_example(cuda):
    from paper_2508_05990_b200 import fme, frame_select as fs
    _, st = fs.open_gop(0, 2, 2, 16)
    kinds = []
    for i in range(1, 4):
        e = np.full((2, 2), 0.4)
        field = fme.MotionField(16, 2, 2, np.zeros((2, 2, 2), np.int64), e, np.ones((2, 2), bool))
        d, st = fs.decide(st, field, i, aem_threshold=1.0)
        kinds.append(d.kind.value)
    assert kinds == ["nonkey_prev_ref", "nonkey_prev_ref", "key"]


def _run_both(clip, labels, pcfg, bayer=True):
    from paper_2508_05990_b200 import pipeline, synth
    frames = synth.frames_of(clip) if bayer else [
        __import__("paper_2508_05990_b200.frame_io", fromlist=["Frame"]).Frame(c.shape[1], c.shape[0], c) for c in clip]
    res = pipeline.run_sequence(frames, {i: l for i, l in enumerate(labels)}, pcfg)
    olab, odec, _ = O.run_sequence(list(clip), bayer, [l.classes for l in labels], ocfg(pcfg.fme),
                                   pcfg.deviation_threshold, pcfg.aem_threshold, pcfg.max_gop, pcfg.aem_statistic,
                                   pcfg.reference_policy)
    for d, (k, r, trig) in zip(res.decisions, odec):
        assert d.kind.value == k and d.reference_index == r and d.trigger_statistic == trig
    for l, ol in zip(res.labels, olab):
        np.testing.assert_array_equal(l.classes, ol)
    return res


def test_pipeline_c1(cuda):
    """Config C1: 256x256 RGGB, 8 frames, v=(2,2), b16 full +-8."""
    from paper_2508_05990_b200 import synth
    from paper_2508_05990_b200.config import PipelineConfig
    from paper_2508_05990_b200.fme import FmeConfig, SearchStage
    clip = synth.bayer_pan_clip(256, 256, 8, (2, 2), seed=3)
    labels = synth.block_labels(256, 256, 8)
    fcfg = FmeConfig(stages=(SearchStage(8, 1), SearchStage(0, 1), SearchStage(0, 1)), block_sizes=(16,))
    _run_both(clip, labels, PipelineConfig(fme=fcfg, refine_enabled=False))


@pytest.mark.parametrize("variant", ["default", "gop5", "mean", "keyframe", "odd_square"])
def test_pipeline_c5_variants(cuda, variant):
    """C5-style: standard preset, moving square, scene cut, decision variants (reduced size)."""
    from paper_2508_05990_b200 import synth
    from paper_2508_05990_b200.config import PipelineConfig
    from paper_2508_05990_b200.fme import get_preset
    w, h, t = 320, 256, 10
    clip = synth.bayer_pan_clip(w, h, t, (6, -4) if variant != "odd_square" else (3, 5), seed=8, square=48,
                                square_velocity=(7, 3))
    clip[7:] = synth.bayer_pan_clip(w, h, t - 7, (2, 2), seed=99)  # scene cut at frame 7
    labels = synth.block_labels(w, h, t)
    kw = dict(fme=get_preset("standard"), refine_enabled=False)
    if variant == "gop5":
        kw.update(max_gop=5, aem_threshold=float("inf"))
    if variant == "mean":
        kw.update(aem_statistic="mean", aem_threshold=0.05)
    if variant == "keyframe":
        kw.update(reference_policy="keyframe")
    res = _run_both(clip, labels, PipelineConfig(**kw))
    if variant == "gop5":
        assert [d.kind.value for d in res.decisions].count("key") == 2


def test_clip_engine_multistream(cuda):
    from paper_2508_05990_b200 import synth
    from paper_2508_05990_b200.config import PipelineConfig
    from paper_2508_05990_b200.engine import ClipEngine
    from paper_2508_05990_b200.fme import FmeConfig, SearchStage
    fcfg = FmeConfig(stages=(SearchStage(4, 1), SearchStage(0, 1), SearchStage(1, 1)), block_sizes=(16,))
    pcfg = PipelineConfig(fme=fcfg, refine_enabled=False)
    S, T, h, w = 3, 5, 96, 128
    clips = np.stack([synth.bayer_pan_clip(w, h, T, (2 * s, -2), seed=50 + s) for s in range(S)])
    eng = ClipEngine(pcfg, h, w, T, S)
    eng.load_frames(clips)
    labels = [synth.block_labels(w, h, T, seed=s) for s in range(S)]
    for s in range(S):
        for t in range(T):
            eng.key_labels[s, t].copy_(cuda.from_numpy(labels[s][t].classes))
    eng.capture()
    eng.replay()
    cuda.cuda.synchronize()
    kinds, refs, trig = eng.decisions_host()
    mv, en, _ = eng.refined_host()
    for s in range(S):
        olab, odec, ofields = O.run_sequence(list(clips[s]), True, [l.classes for l in labels[s]], ocfg(fcfg))
        for t in range(1, T):
            p = eng.pair_index(s, t)
            np.testing.assert_array_equal(mv[p], ofields[t][1].mv)
            np.testing.assert_array_equal(en[p].view(np.int64), ofields[t][1].energy.view(np.int64))
            assert odec[t][0] == ("key", "nonkey_prev_ref", "nonkey_key_ref")[kinds[s, t]]
            assert trig[s, t] == odec[t][2]
        got = eng.labels[s].cpu().numpy()
        for t in range(T):
            np.testing.assert_array_equal(got[t], olab[t])


@pytest.mark.parametrize("variant", ["callable", "tensor", "gop3", "keyframe", "ringvote", "ringvote_tensor"])
def test_clip_session_matches_run_sequence(cuda, variant):
    """The pipelined host-buffer session (chunked H2D / ME / label chain / D2H on three
    streams) returns exactly what run_sequence returns, for both key-label forms."""
    from paper_2508_05990_b200 import synth
    from paper_2508_05990_b200.config import PipelineConfig
    from paper_2508_05990_b200.fme import FmeConfig, SearchStage
    from paper_2508_05990_b200.pipeline import ClipSession, run_sequence
    w, h, t = 192, 128, 11
    clip = synth.bayer_pan_clip(w, h, t, (4, -2), seed=21, square=32, square_velocity=(5, 3))
    labels = synth.block_labels(w, h, t, seed=4)
    fcfg = FmeConfig(stages=(SearchStage(4, 1), SearchStage(0, 1), SearchStage(1, 1)), block_sizes=(16,))
    kw = dict(fme=fcfg, refine_enabled=variant.startswith("ringvote"), aem_threshold=0.02)
    if variant == "gop3" or variant.startswith("ringvote"):
        kw.update(max_gop=3, aem_threshold=float("inf"))
    if variant == "keyframe":
        kw.update(reference_policy="keyframe")
    pcfg = PipelineConfig(**kw)
    ref = run_sequence(synth.frames_of(clip), labels, pcfg)
    sess = ClipSession(pcfg, h, w, t, np.uint8, True, chunks=3)
    if variant.endswith("tensor"):
        key = cuda.from_numpy(np.stack([l.classes for l in labels])).pin_memory()
    else:
        key = {i: labels[i] for i in range(t)}
    for _ in range(2):  # a second run on the same session must not see stale state
        got, kinds, refs, trig = sess.run(cuda.from_numpy(clip).pin_memory(), key)
        for i, d in enumerate(ref.decisions):
            assert ("key", "nonkey_prev_ref", "nonkey_key_ref")[kinds[i]] == d.kind.value
            assert trig[i] == d.trigger_statistic
            if kinds[i] != 0:
                assert refs[i] == d.reference_index
        for i in range(t):
            np.testing.assert_array_equal(got[i], ref.labels[i].classes)


def test_ring_vote_pipeline_matches_oracle(cuda):
    """run_sequence with the default refine_enabled (no CaBR weights): the flagged blocks of every
    predicted frame take CaBR's ring vote and the refined labels feed later predictions."""
    from paper_2508_05990_b200 import synth
    from paper_2508_05990_b200.config import PipelineConfig
    from paper_2508_05990_b200.fme import FmeConfig, SearchStage
    from paper_2508_05990_b200.pipeline import run_sequence
    w, h, t = 224, 160, 7
    clip = synth.bayer_pan_clip(w, h, t, (5, -3), seed=13, square=48, square_velocity=(9, 5))
    labels = synth.block_labels(w, h, t, seed=9)
    fcfg = FmeConfig(stages=(SearchStage(3, 1), SearchStage(0, 1), SearchStage(1, 1)), block_sizes=(16, 8))
    pcfg = PipelineConfig(fme=fcfg, max_gop=5, aem_threshold=float("inf"))
    res = run_sequence(synth.frames_of(clip), labels, pcfg)
    olab, odec, _ = O.run_sequence(list(clip), True, [l.classes for l in labels], ocfg(fcfg), pcfg.deviation_threshold,
                                   pcfg.aem_threshold, pcfg.max_gop, ring_vote=True)
    assert [d.kind.value for d in res.decisions] == [k for k, _, _ in odec]
    for i in range(t):
        np.testing.assert_array_equal(res.labels[i].classes, olab[i])


@pytest.mark.parametrize("policy", ["previous", "keyframe"])
def test_multistream_engine_ring_vote(cuda, policy):
    """Three streams in one engine with CaBR's ring vote in the label chain == the oracle per stream."""
    from paper_2508_05990_b200 import synth
    from paper_2508_05990_b200.config import PipelineConfig
    from paper_2508_05990_b200.engine import ClipEngine
    from paper_2508_05990_b200.fme import FmeConfig, SearchStage
    fcfg = FmeConfig(stages=(SearchStage(3, 1), SearchStage(0, 1), SearchStage(1, 1)), block_sizes=(16,))
    pcfg = PipelineConfig(fme=fcfg, max_gop=4, aem_threshold=float("inf"), reference_policy=policy)
    S, T, h, w = 3, 6, 128, 160
    clips = np.stack([synth.bayer_pan_clip(w, h, T, (2 * s + 1, -3), seed=70 + s, square=32,
                                           square_velocity=(5, 2 * s)) for s in range(S)])
    eng = ClipEngine(pcfg, h, w, T, S)
    eng.load_frames(clips)
    labels = [synth.block_labels(w, h, T, seed=s) for s in range(S)]
    for s in range(S):
        for t in range(T):
            eng.key_labels[s, t].copy_(cuda.from_numpy(labels[s][t].classes.copy()))
    eng.step()
    cuda.cuda.synchronize()
    for s in range(S):
        olab, _, _ = O.run_sequence(list(clips[s]), True, [l.classes for l in labels[s]], ocfg(fcfg),
                                    pcfg.deviation_threshold, pcfg.aem_threshold, pcfg.max_gop,
                                    reference_policy=policy, ring_vote=True)
        got = eng.labels[s].cpu().numpy()
        for t in range(T):
            np.testing.assert_array_equal(got[t], olab[t])


# ---------------------------------------------------------------------------
# float64 plane stacks (fme.py:188-190) and geometry outside the integer kernels
# ---------------------------------------------------------------------------

F64_CASES = [
    # (P, h, w, block_sizes, stages, value range)
    (4, 72, 96, (16, 8), ((3, 2), (1, 1), (1, 1)), 1.0),
    (3, 64, 48, (16,), ((4, 1), (0, 1), (2, 1)), 0.2),
    (1, 50, 70, (32, 16, 8), ((2, 4), (1, 2), (1, 1)), 3.0),
    (4, 40, 40, (8,), ((2, 1), (1, 1), (1, 1)), 1e-3),
]


@pytest.mark.parametrize("case", range(len(F64_CASES)))
def test_estimate_motion_float_stacks(cuda, case):
    from paper_2508_05990_b200 import fme, mv_refine
    from paper_2508_05990_b200.fme import FmeConfig, SearchStage
    P, h, w, bs, stages, hi = F64_CASES[case]
    rng = np.random.default_rng(100 + case)
    cur = rng.random((P, h, w)) * hi
    ref = np.roll(cur, (1, -2), axis=(1, 2)) + rng.random((P, h, w)) * hi * 0.05
    if case == 3:  # quantised values -> many exact ties
        cur, ref = np.round(cur * 3e3) / 3e3, np.round(ref * 3e3) / 3e3
    cfg = FmeConfig(stages=tuple(SearchStage(*s) for s in stages), block_sizes=bs, lam=0.3,
                    sparsity_tolerance=0.01 * hi if hi <= 1 else 0.03)
    c2, r2 = (cur[0], ref[0]) if P == 1 else (cur, ref)  # a 2-D ndarray is a one-plane stack
    got = fme.estimate_motion(c2, r2, cfg)
    want = O.estimate_motion(cur, ref, ocfg(cfg))
    assert_levels_equal(got, want)
    r_got = mv_refine.refine_mvs(got[-1], 1, cur=c2, ref=r2, config=cfg)
    r_want = O.refine_mvs(want[-1], 1, cur, ref, ocfg(cfg))
    np.testing.assert_array_equal(r_got.mv, r_want.mv)
    np.testing.assert_array_equal(r_got.energy.view(np.int64), r_want.energy.view(np.int64))


def test_estimate_motion_block_128_frames(cuda):
    """FmeConfig admits any power-of-two block >= 8 (fme.py:65-67); 128 goes through
    the float64 kernel on device-normalised planes, bit-exact."""
    from paper_2508_05990_b200 import fme, synth
    from paper_2508_05990_b200.fme import FmeConfig, SearchStage
    clip = synth.bayer_pan_clip(600, 520, 2, (6, -4), seed=8)
    fr = synth.frames_of(clip)
    cfg = FmeConfig(stages=(SearchStage(2, 4), SearchStage(1, 2), SearchStage(1, 1)), block_sizes=(128, 64))
    got = fme.estimate_motion(fr[1], fr[0], cfg)
    want = O.estimate_motion(O.search_planes(clip[1], True), O.search_planes(clip[0], True), ocfg(cfg))
    assert_levels_equal(got, want)


@pytest.mark.parametrize("bsize", [5, 12, 3])
def test_search_stage_any_block_size(cuda, bsize):
    from paper_2508_05990_b200 import fme
    from paper_2508_05990_b200.frame_io import Frame, FrameKind
    cfg = _cfgs()["lam0"]
    rng = np.random.default_rng(bsize)
    a = rng.integers(0, 256, (40, 44)).astype(np.uint8)
    b = np.roll(a, (2, 1), axis=(0, 1))
    for cur, ref, planes_c, planes_r in (
            (Frame(44, 40, a, FrameKind.LUMA), Frame(44, 40, b, FrameKind.LUMA),
             O.search_planes(a, False), O.search_planes(b, False)),
            (a / 7.0, b / 7.0, (a / 7.0)[None], (b / 7.0)[None])):
        for origin, center in (((10, 9), (0, 0)), ((0, 0), (-1, 2)), ((44 - bsize, 40 - bsize), (3, 3))):
            got = fme.search_stage(cur, ref, origin, bsize, center, 3, 1, cfg)
            mv, e, _ = O.stage_candidates(planes_r, planes_c[:, origin[1]:origin[1] + bsize,
                                                             origin[0]:origin[0] + bsize],
                                          origin, bsize, center, 3, 1, cfg.lam, cfg.sparsity_tolerance)
            assert got[0] == tuple(mv) and np.float64(got[1]).view(np.int64) == np.float64(e).view(np.int64)
    with pytest.raises(ValueError, match="all candidate windows fall outside"):
        fme.search_stage(a / 1.0, b / 1.0, (0, 0), bsize, (-30, -30), 1, 1, cfg)


@pytest.mark.parametrize("max_gop", [None, 4])
@pytest.mark.parametrize("policy", ["previous", "keyframe"])
def test_decide_large_grid_parallel_scan(cuda, max_gop, policy):
    """AEM scans over accumulator grids too large for the register-resident kernel take the
    parallel form (maxima of every reset point, then a serial scan): per-frame calls and one
    call over a frame range, split in two resumable calls, all equal the oracle bit for bit."""
    import ctypes
    from paper_2508_05990_b200 import _native as N, fme, frame_select as fs
    rng = np.random.default_rng(23)
    for (ch, cw, f) in [(90, 120, 1), (60, 70, 2)]:
        T = 14
        es = [rng.random((ch * f, cw * f)) * 0.03 for _ in range(T)]
        # oracle
        acc, fsk, last_key = np.zeros((ch, cw)), 0, 0
        want = []
        for i in range(1, T):
            kind, ref, trig, acc, fsk = O.decide(acc, fsk, 32, es[i], 32 // f, i, 0.15, max_gop, "max", policy, last_key)
            want.append((kind, ref, trig))
            if kind == "key":
                last_key = i
        # per-frame drop-in calls
        st = fs.AemState.fresh(cw, ch, 32)
        lk = 0
        for i in range(1, T):
            field = fme.MotionField(32 // f, cw * f, ch * f, np.zeros((ch * f, cw * f, 2), np.int64), es[i],
                                    np.ones_like(es[i], bool))
            d, st = fs.decide(st, field, i, 0.15, max_gop, "max", policy, lk)
            assert (d.kind.value, d.reference_index, d.trigger_statistic) == want[i - 1]
            if d.kind.value == "key":
                lk = i
        np.testing.assert_array_equal(st.accumulated, acc)
        # frame-range calls straight through the C ABI, split at frame 6
        dev = cuda.device("cuda")
        e = cuda.from_numpy(np.stack(es)).to(dev)
        sp = N.select_params(ch * f, cw * f, f, ch, cw, "max", policy, max_gop, 0.15)
        accd = cuda.zeros((ch, cw), dtype=cuda.float64, device=dev)
        fskd = cuda.zeros(1, dtype=cuda.int32, device=dev)
        lkd = cuda.zeros(1, dtype=cuda.int32, device=dev)
        kind = cuda.zeros(T, dtype=cuda.int32, device=dev)
        ref = cuda.full((T,), -1, dtype=cuda.int32, device=dev)
        trig = cuda.zeros(T, dtype=cuda.float64, device=dev)
        cells = ch * f * cw * f
        for t0, t1 in ((1, 6), (6, T)):
            N.check(N.load().bmc_decide(N.ptr(e), cells, cells, 1, t0, t1, ctypes.byref(sp), N.ptr(accd), N.ptr(fskd),
                                        N.ptr(lkd), N.ptr(kind), N.ptr(ref), N.ptr(trig), T, None, T,
                                        N.stream_handle()))
        k, r, tr = kind.cpu().numpy(), ref.cpu().numpy(), trig.cpu().numpy()
        names = ["key", "nonkey_prev_ref", "nonkey_key_ref"]
        for i in range(1, T):
            assert (names[k[i]], None if r[i] < 0 else int(r[i]), float(tr[i])) == want[i - 1]
        np.testing.assert_array_equal(accd.cpu().numpy(), acc)


def test_clip_pool_matches_sessions(cuda):
    """ClipPool (two sessions on their own streams, one host thread each) equals one
    ClipSession run per clip, in input order."""
    from paper_2508_05990_b200 import pipeline, synth
    from paper_2508_05990_b200.config import PipelineConfig
    from paper_2508_05990_b200.fme import FmeConfig, SearchStage
    cfg = PipelineConfig(fme=FmeConfig(stages=(SearchStage(8, 1), SearchStage(0, 1), SearchStage(0, 1)),
                                       block_sizes=(16,)), max_gop=3, aem_threshold=float("inf"))
    clips, keys = [], []
    for k in range(5):
        c = synth.bayer_pan_clip(256, 192, 7, (2 * (k % 3) - 2, 2), seed=40 + k)
        clips.append(cuda.from_numpy(c).pin_memory())
        keys.append(cuda.from_numpy(np.stack([l.classes for l in synth.block_labels(256, 192, 7, seed=k)])).pin_memory())
    pool = pipeline.ClipPool(cfg, 192, 256, 7, np.uint8, True, n_sessions=2)
    got = pool.run(list(zip(clips, keys)))
    sess = pipeline.ClipSession(cfg, 192, 256, 7, np.uint8, True)
    for (raw, key), g in zip(zip(clips, keys), got):
        want = sess.run(raw, key)
        for a, b in zip(g[0], want[0]):
            np.testing.assert_array_equal(a, b)
        np.testing.assert_array_equal(g[1], want[1])
        np.testing.assert_array_equal(g[2], want[2])
