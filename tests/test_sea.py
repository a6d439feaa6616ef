"""GPU: the successive-elimination (SEA) screening of unit-step ME stages
(csrc/bmc_fme_impl.cuh sea_screen) against the oracle, bit-exact, on the
content that decides which path a block takes:

* exact translations (a zero-SAD match per interior block: SEA settles the block),
  uint8 and uint16 Bayer, luma (one plane);
* several zero-SAD candidates (periodic texture): the FIRST in canonical
  dy-major order must win (np.argmin, fme.py:266);
* flat frames (every bound 0, every SAD 0): too many survivors, dense fallback;
* noise (no exact match): dense fallback;
* lam = 1 (SEA disabled: energy ties without SAD ties);
* kblk pairs where one block has an exact match and its neighbour does not.
"""

import numpy as np
import pytest

from oracle import bayermc_oracle as O

pytestmark = pytest.mark.gpu


def _levels_equal(got, want):
    assert len(got) == len(want)
    for g, o in zip(got, want):
        np.testing.assert_array_equal(g.mv, o.mv)
        np.testing.assert_array_equal(g.matched, o.matched)
        assert g.candidate_evals == o.candidate_evals
        np.testing.assert_array_equal(g.energy.view(np.int64), o.energy.view(np.int64))


def _run(cur, ref, bayer, cfg):
    from paper_2508_05990_b200 import fme
    from paper_2508_05990_b200.frame_io import Frame, FrameKind
    kind = FrameKind.BAYER_RGGB if bayer else FrameKind.LUMA
    h, w = cur.shape
    got = fme.estimate_motion(Frame(w, h, cur, kind), Frame(w, h, ref, kind), cfg)
    oc = O.cfg_dict(stages=[(s.range, s.step) for s in cfg.stages], lam=cfg.lam, block_sizes=cfg.block_sizes,
                    split_threshold=cfg.split_threshold, sparsity_tolerance=cfg.sparsity_tolerance,
                    refine_block_threshold=cfg.refine_block_threshold)
    want = O.estimate_motion(O.search_planes(cur, bayer), O.search_planes(ref, bayer), oc)
    _levels_equal(got, want)
    return got


def _full(r=8, b=16, lam=0.1):
    from paper_2508_05990_b200.fme import FmeConfig, SearchStage
    return FmeConfig(stages=(SearchStage(r, 1), SearchStage(0, 1), SearchStage(0, 1)), block_sizes=(b,), lam=lam)


@pytest.mark.parametrize("dtype,bayer", [(np.uint8, True), (np.uint16, True), (np.uint8, False)])
def test_sea_exact_translation(cuda, dtype, bayer):
    from paper_2508_05990_b200 import synth
    clip = synth.bayer_pan_clip(192, 160, 2, (4, -2), seed=21, dtype=dtype)
    got = _run(clip[1], clip[0], bayer, _full())
    assert (got[-1].energy == 0).mean() > 0.5  # most blocks found their exact match


def test_sea_first_of_several_zero_sad_candidates(cuda):
    # a texture periodic with 6 plane pixels (12 raw): every interior block has
    # exact matches 6 apart, and block sums (16 is not a multiple of 6) still
    # differ between most candidates, so SEA settles the blocks itself
    rng = np.random.default_rng(5)
    tile = rng.integers(0, 256, (12, 12), dtype=np.uint8)
    big = np.tile(tile, (16, 20))
    cur, ref = big[:160, 12:204].copy(), big[:160, :192].copy()
    got = _run(cur, ref, True, _full())
    assert (got[-1].energy == 0).all()
    assert (got[-1].mv[2:-2, 2:-2] == -6).all()  # the first (dy, dx) = (-6, -6) in canonical order


def test_sea_flat_frames_fall_back(cuda):
    cur = np.full((128, 160), 77, np.uint8)
    got = _run(cur, cur.copy(), True, _full())
    assert (got[-1].mv[..., 0] == -8).sum() > 0  # first valid candidate in canonical order wins ties


def test_sea_noise_falls_back(cuda):
    rng = np.random.default_rng(9)
    cur = rng.integers(0, 256, (128, 160), dtype=np.uint8)
    ref = rng.integers(0, 256, (128, 160), dtype=np.uint8)
    _run(cur, ref, True, _full())


def test_sea_lam1_is_dense(cuda):
    from paper_2508_05990_b200 import synth
    clip = synth.bayer_pan_clip(128, 128, 2, (2, 2), seed=4)
    _run(clip[1], clip[0], True, _full(r=6, lam=1.0))


def test_sea_mixed_kblk_pair(cuda):
    # left half translated exactly, right half fresh noise: CTAs pairing one block of each
    from paper_2508_05990_b200 import synth
    clip = synth.bayer_pan_clip(256, 128, 2, (2, 0), seed=13)
    rng = np.random.default_rng(3)
    cur = clip[1].copy()
    cur[:, 112:] = rng.integers(0, 256, (128, 144), dtype=np.uint8)
    _run(cur, clip[0], True, _full(r=16))


def test_sea_pipeline_matches_oracle(cuda):
    """run_sequence over a pan clip with a moving square (SEA and dense blocks mixed)."""
    from paper_2508_05990_b200 import pipeline, synth
    from paper_2508_05990_b200.config import PipelineConfig
    clip = synth.bayer_pan_clip(256, 192, 5, (4, 2), seed=17, square=48, square_velocity=(6, -2))
    labels = synth.block_labels(256, 192, 5)
    cfg = PipelineConfig(fme=_full(r=12), refine_enabled=False, max_gop=4, aem_threshold=float("inf"))
    frames = synth.frames_of(clip)
    res = pipeline.run_sequence(frames, {i: l for i, l in enumerate(labels)}, cfg)
    want, decs, _ = O.run_sequence(list(clip), True, [l.classes for l in labels], O.cfg_dict(
        stages=[(12, 1), (0, 1), (0, 1)], block_sizes=(16,)), max_gop=4, aem_threshold=float("inf"))
    for g, w in zip(res.labels, want):
        np.testing.assert_array_equal(g.classes, w)
    assert [d.trigger_statistic for d in res.decisions] == [t for _, _, t in decs]
