"""CPU: host-side logic of the drop-in modules (types, validation messages,
presets, JSON, FLOP counters, synthetic clips, config loader) and the
no-fallback contract (compute entry points raise without CUDA)."""

import numpy as np
import pytest

from paper_2508_05990_b200 import config, fme, frame_io, frame_select, metrics, mv_refine, propagate, synth


def test_fmeconfig_validation_messages():
    S = fme.SearchStage
    with pytest.raises(ValueError, match="exactly three search stages"):
        fme.FmeConfig(stages=(S(1, 1),))
    with pytest.raises(ValueError, match="power of two >= 8"):
        fme.FmeConfig(block_sizes=(24,))
    with pytest.raises(ValueError, match="sizes must halve"):
        fme.FmeConfig(block_sizes=(64, 16))
    with pytest.raises(ValueError, match="lambda weight"):
        fme.FmeConfig(lam=1.5)
    with pytest.raises(ValueError, match="split_threshold must be in"):
        fme.FmeConfig(split_threshold=-0.1)
    with pytest.raises(ValueError, match="search range must be >= 0"):
        S(-1, 1)
    with pytest.raises(ValueError, match="search step must be >= 1"):
        S(1, 0)
    with pytest.raises(ValueError, match="unknown preset"):
        fme.get_preset("nope")


def test_presets_match_reference_table3(reference):
    from bayermc import fme as RF
    assert set(fme.PRESETS) == set(RF.PRESETS)
    for k in fme.PRESETS:
        a, b = fme.PRESETS[k], RF.PRESETS[k]
        assert [(s.range, s.step) for s in a.stages] == [(s.range, s.step) for s in b.stages]
        assert (a.lam, a.block_sizes, a.split_threshold, a.sparsity_tolerance, a.refine_block_threshold) == \
               (b.lam, b.block_sizes, b.split_threshold, b.sparsity_tolerance, b.refine_block_threshold)


def test_flop_counters_match_reference(reference):
    from bayermc import fme as RF, mv_refine as RM
    assert fme.flops_per_candidate(64) == 12291
    std = fme.get_preset("standard")
    assert fme.count_fme_flops((2048, 1024), std, 512 * 131) == RF.count_fme_flops((2048, 1024), RF.get_preset(
        "standard"), 512 * 131)
    assert abs(fme.count_fme_flops((2048, 1024), std, 512 * 131) / 1e9 - 0.824) < 1e-3
    for gw, gh, b, rep, P in [(60, 34, 16, 5, 4), (1, 1, 8, 0, 1), (2, 7, 32, 3, 1), (15, 9, 64, 1, 4)]:
        assert mv_refine.count_refine_flops(gw, gh, b, rep, P) == RM.count_refine_flops(gw, gh, b, rep, P)
    with pytest.raises(ValueError):
        fme.count_fme_flops((64, 64), std, [1])


def test_motion_field_json_roundtrip(tmp_path):
    mv = np.arange(24).reshape(3, 4, 2)
    f = fme.MotionField(16, 4, 3, mv, np.linspace(0, 1, 12).reshape(3, 4), np.eye(3, 4, dtype=bool), 1, 77)
    fme.save_motion_field([f, f], tmp_path / "f.json")
    g = fme.load_motion_field(tmp_path / "f.json")
    np.testing.assert_array_equal(g.mv, f.mv)
    np.testing.assert_array_equal(g.energy, f.energy)
    np.testing.assert_array_equal(g.matched, f.matched)
    assert f.refinement_blocks() == [(x, y) for y in range(3) for x in range(4) if not (x == y)]
    assert not f.mv.flags.writeable
    with pytest.raises(ValueError, match="mv must have shape"):
        fme.MotionField(16, 4, 3, mv[:, :3], f.energy, f.matched)


def test_frame_types_and_cfa():
    d = np.arange(16, dtype=np.uint8).reshape(4, 4)
    f = frame_io.Frame(4, 4, d, frame_io.FrameKind.BAYER_RGGB)
    planes = frame_io.pack_bayer(f).planes
    assert [p.ravel().tolist() for p in planes] == [[0, 2, 8, 10], [1, 3, 9, 11], [4, 6, 12, 14], [5, 7, 13, 15]]
    np.testing.assert_array_equal(frame_io.unpack_bayer(frame_io.pack_bayer(f)).data, d)
    with pytest.raises(ValueError, match="even width and height"):
        frame_io.Frame(3, 4, np.zeros((4, 3), np.uint8), frame_io.FrameKind.BAYER_GBRG)
    with pytest.raises(ValueError, match="uint8 or uint16"):
        frame_io.Frame(2, 2, np.zeros((2, 2), np.float32))
    with pytest.raises(ValueError, match="requires a Bayer frame"):
        frame_io.pack_bayer(frame_io.Frame(2, 2, np.zeros((2, 2), np.uint8)))
    r, g, b = (np.full((2, 2), v, np.uint8) for v in (200, 100, 50))
    m = frame_io.mosaic_rgb(r, g, b, frame_io.FrameKind.BAYER_RGGB).data
    assert m.tolist() == [[200, 100], [100, 50]]
    with pytest.raises(ValueError, match="class ID"):
        frame_io.LabelMap(2, 2, np.full((2, 2), 3, np.uint8), 3)


def test_synthetic_clip_recipe_matches_reference_noise(reference):
    from bayermc import synth as RS
    for args in [(100, 60, 3, 16), (257, 33, 9, 8)]:
        np.testing.assert_array_equal(synth.value_noise(*args), RS.value_noise(*args))
    clip = synth.bayer_pan_clip(64, 48, 3, (2, -2), seed=1)
    # even velocities keep CFA phase: frame t+1 plane-shifted by v/2
    p0 = np.stack(frame_io.pack_bayer(frame_io.Frame(64, 48, clip[0], frame_io.FrameKind.BAYER_RGGB)).planes)
    p1 = np.stack(frame_io.pack_bayer(frame_io.Frame(64, 48, clip[1], frame_io.FrameKind.BAYER_RGGB)).planes)
    np.testing.assert_array_equal(p1[:, 1:-1, 0:-2], p0[:, 0:-2, 1:-1])


def test_pipeline_config_toml(tmp_path):
    p = tmp_path / "c.toml"
    p.write_text('[fme]\npreset = "mode1"\nlambda = 0.3\n[frame_select]\nmax_gop = 5\nstatistic = "mean"\n'
                 'reference = "keyframe"\n[cabr]\nenabled = false\n')
    c = config.load_pipeline_config(p)
    assert c.fme.lam == 0.3 and c.fme.stages[0].range == 6 and c.max_gop == 5
    assert (c.aem_statistic, c.reference_policy, c.refine_enabled) == ("mean", "keyframe", False)
    assert config.load_pipeline_config(preset="mode3").fme.block_sizes == (32,)


def test_flop_ledger():
    L = metrics.FlopLedger()
    L.add("fme", 10)
    L.add("prediction", 0)
    with pytest.raises(ValueError, match="stays 0"):
        L.add("prediction", 1)
    with pytest.raises(ValueError, match="unknown component"):
        L.add("x", 1)
    assert metrics.FlopLedger.from_json(L.to_json()).as_dict() == L.as_dict()
    assert "total" in L.table()


def test_decision_types():
    d, st = frame_select.open_gop(0, 3, 2, 64)
    assert d.kind is frame_select.DecisionKind.KEY and st.accumulated.shape == (2, 3)
    with pytest.raises(ValueError, match="open_gop only applies"):
        frame_select.open_gop(1, 3, 2, 64)
    with pytest.raises(ValueError, match="earlier reference"):
        frame_select.FrameDecision(3, frame_select.DecisionKind.NONKEY_PREV_REF, 3)
    assert frame_select.kind_from_code(2) is frame_select.DecisionKind.NONKEY_KEY_REF


def test_no_cpu_fallback(monkeypatch):
    """Compute entry points must fail loudly when CUDA is unavailable."""
    import torch
    monkeypatch.setattr(torch.cuda, "is_available", lambda: False)
    f = frame_io.Frame(32, 32, np.zeros((32, 32), np.uint8))
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        fme.estimate_motion(f, f, fme.FmeConfig(block_sizes=(16,)))
    fld = fme.MotionField(16, 2, 2, np.zeros((2, 2, 2), np.int64), np.zeros((2, 2)), np.ones((2, 2), bool))
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        mv_refine.refine_mvs(fld)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        propagate.predict_labels(frame_io.LabelMap(32, 32, np.zeros((32, 32), np.uint8), 2), fld)
    _, st = frame_select.open_gop(0, 2, 2, 16)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        frame_select.decide(st, fld, 1)


def test_validation_precedes_device(monkeypatch):
    """Reference error messages are raised before any device work."""
    f = frame_io.Frame(32, 32, np.zeros((32, 32), np.uint8))
    g = frame_io.Frame(32, 32, np.zeros((32, 32), np.uint8), frame_io.FrameKind.BAYER_RGGB)
    with pytest.raises(ValueError, match="frame kind mismatch"):
        fme.estimate_motion(f, g)
    fld = fme.MotionField(16, 1, 1, np.zeros((1, 1, 2), np.int64), np.zeros((1, 1)), np.ones((1, 1), bool))
    with pytest.raises(ValueError, match="scale must be 1 or 2"):
        propagate.predict_labels(frame_io.LabelMap(8, 8, np.zeros((8, 8), np.uint8), 2), fld, 3)
    with pytest.raises(ValueError, match="motion field covers"):
        propagate.predict_labels(frame_io.LabelMap(80, 8, np.zeros((8, 80), np.uint8), 2), fld, 1)
    with pytest.raises(TypeError):
        propagate.predict_labels(frame_io.LabelMap(8, 8, np.zeros((8, 8), np.uint8), 2), "x")
    _, st = frame_select.open_gop(0, 1, 1, 16)
    with pytest.raises(ValueError, match="statistic must be"):
        frame_select.decide(st, fld, 1, statistic="median")
    fld2 = fme.MotionField(32, 1, 1, np.zeros((1, 1, 2), np.int64), np.zeros((1, 1)), np.ones((1, 1), bool))
    with pytest.raises(ValueError, match="does not divide"):
        frame_select.decide(st, fld2, 1)


def test_bench_config_table():
    import bench
    assert bench.CONFIGS["c2"][:3] == (1920, 1080, 30)
    pc = bench.pipeline_config("c2")
    assert pc.fme.block_sizes == (16,) and pc.fme.stages[0].range == 16 and not pc.refine_enabled
