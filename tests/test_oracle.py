"""CPU: pin the oracle against the reference's own outputs (golden fixtures made
by tests/golden/make_golden.py) and, when /root/reference is mounted, against
the live reference on fresh seeded inputs."""

import numpy as np
import pytest

import golden_io as G
from oracle import bayermc_oracle as O


def bits(a):
    return np.asarray(a, dtype=np.float64).view(np.int64)


@pytest.mark.parametrize("name", G.me_fixture_names())
def test_oracle_matches_golden_me(name):
    d = G.load(name)
    bayer = bool(d["bayer"])
    got = O.estimate_motion(O.search_planes(d["cur"], bayer), O.search_planes(d["ref"], bayer), G.oracle_cfg(d))
    want = G.levels(d)
    assert len(got) == len(want)
    for g, (mv, en, matched, evals, b) in zip(got, want):
        assert g.block_size == b
        np.testing.assert_array_equal(g.mv, mv)
        np.testing.assert_array_equal(bits(g.energy), bits(en))
        np.testing.assert_array_equal(g.matched, matched)
        assert g.candidate_evals == evals


@pytest.mark.parametrize("name", G.pipe_fixture_names())
def test_oracle_matches_golden_pipeline(name):
    d = G.load(name)
    clip, keys = G.pipe_inputs(d)
    pc = G.pipeline_config(d)
    labels, dec, _ = O.run_sequence(list(clip), True, list(keys), G.oracle_cfg(d), pc.deviation_threshold,
                                    pc.aem_threshold, pc.max_gop, pc.aem_statistic, pc.reference_policy,
                                    ring_vote=pc.refine_enabled)
    codes = {"key": 0, "nonkey_prev_ref": 1, "nonkey_key_ref": 2}
    np.testing.assert_array_equal([codes[k] for k, _, _ in dec], d["kinds"])
    np.testing.assert_array_equal([-1 if r is None else r for _, r, _ in dec], d["refs"])
    np.testing.assert_array_equal(bits([t for _, _, t in dec]), bits(d["trig"]))
    np.testing.assert_array_equal(np.stack(labels), d["out_labels"])


def test_oracle_kats():
    k = G.load("kats.npz")
    a = np.zeros((64, 64))
    b = a.copy()
    b[3, 5] = 0.2
    assert O.block_energy(a, b, 0.1, 8 / 255) == float(k["kat_block_energy"])
    assert abs(float(k["kat_block_energy"]) - 6.8359375e-05) < 1e-12
    raw = np.arange(16, dtype=np.uint8).reshape(4, 4)
    np.testing.assert_array_equal(np.stack(O.pack_bayer(raw)), k["kat_pack_bayer"])
    np.testing.assert_array_equal(k["kat_pack_bayer"].reshape(4, 4),
                                  [[0, 2, 8, 10], [1, 3, 9, 11], [4, 6, 12, 14], [5, 7, 13, 15]])
    f = O.OracleField(16, k["kat_refine_in"].copy(), np.zeros((3, 3)), np.ones((3, 3), bool), 0, 0)
    np.testing.assert_array_equal(O.refine_mvs(f, 4).mv, k["kat_refine_out"])
    mvp = k["prop_mv"]
    fld = O.OracleField(16, mvp, np.zeros(mvp.shape[:2]), np.ones(mvp.shape[:2], bool), 0, 0)
    np.testing.assert_array_equal(O.predict_labels(k["prop_in"], fld, 2), k["prop_out"])


def test_oracle_decide_sequences():
    d = G.load("decide_sequences.npz")
    for statistic in ("max", "mean"):
        for max_gop in (None, 3):
            for policy in ("previous", "keyframe"):
                key = f"{statistic}_{max_gop}_{policy}"
                acc, fsk, last_key = np.zeros((9, 15)), 0, 0
                for i, e in enumerate(d[key + "_e"], start=1):
                    kind, ref, trig, acc, fsk = O.decide(acc, fsk, 32, e, 16, i, 0.15, max_gop, statistic, policy,
                                                         last_key)
                    assert kind == d[key + "_kinds"][i - 1]
                    assert (-1 if ref is None else ref) == d[key + "_refs"][i - 1]
                    assert trig == d[key + "_trig"][i - 1]
                    if kind == "key":
                        last_key = i


@pytest.mark.parametrize("n", [1, 5, 7, 8, 64, 100, 127, 128, 129, 255, 256, 1000, 1024, 2040, 4096, 12345, 16384,
                               32400])
def test_pairwise_matches_numpy_sum(n):
    x = np.random.default_rng(n).random((3, n))
    np.testing.assert_array_equal(O.pairwise_sum_rows(x), x.sum(axis=1))
    np.testing.assert_array_equal(O.pairwise_sum_rows(x) / n, np.array([r.mean() for r in x]))


def test_oracle_vs_live_reference(reference):
    """Fresh seeded cases against the live reference (build container only)."""
    from bayermc import fme as F, frame_io as FI, frame_select as FS, mv_refine as MR, propagate as PR
    rng = np.random.default_rng(99)
    cfgs = [F.FmeConfig(), F.FmeConfig(stages=(F.SearchStage(3, 2), F.SearchStage(0, 1), F.SearchStage(1, 1)),
                                       block_sizes=(16, 8), lam=0.25)]
    for trial in range(6):
        h, w = [(64, 96), (128, 128), (70, 54)][trial % 3]
        dt = np.uint16 if trial % 2 else np.uint8
        hi = [7, 256, 60000][trial % 3] if dt == np.uint16 else [7, 256, 40][trial % 3]
        bayer = trial % 3 != 2
        kind = FI.FrameKind.BAYER_RGGB if bayer else FI.FrameKind.LUMA
        a = rng.integers(0, hi, (h, w)).astype(dt)
        b = rng.integers(0, hi, (h, w)).astype(dt)
        for c in cfgs:
            ref = F.estimate_motion(FI.Frame(w, h, a, kind), FI.Frame(w, h, b, kind), c)
            oc = O.cfg_dict(stages=[(s.range, s.step) for s in c.stages], lam=c.lam, block_sizes=c.block_sizes)
            got = O.estimate_motion(O.search_planes(a, bayer), O.search_planes(b, bayer), oc)
            for g, r in zip(got, ref):
                np.testing.assert_array_equal(g.mv, r.mv)
                np.testing.assert_array_equal(bits(g.energy), bits(r.energy))
                np.testing.assert_array_equal(g.matched, r.matched)
                assert g.candidate_evals == r.candidate_evals
            r2 = MR.refine_mvs(ref[-1], 1, cur=FI.Frame(w, h, a, kind), ref=FI.Frame(w, h, b, kind), config=c)
            o2 = O.refine_mvs(got[-1], 1, O.search_planes(a, bayer), O.search_planes(b, bayer), oc)
            np.testing.assert_array_equal(o2.mv, r2.mv)
            np.testing.assert_array_equal(bits(o2.energy), bits(r2.energy))
            lab = rng.integers(0, 5, (h, w)).astype(np.uint8)
            scale = 2 if bayer else 1
            if ref[-1].grid_w * ref[-1].block_size * scale >= w and ref[-1].grid_h * ref[-1].block_size * scale >= h:
                np.testing.assert_array_equal(
                    O.predict_labels(lab, o2, scale),
                    PR.predict_labels(FI.LabelMap(w, h, lab, 5), r2, scale).classes)
    # AEM state machine, mean statistic on an odd-sized grid
    _, st = FS.open_gop(0, 7, 5, 32)
    acc, fsk = np.zeros((5, 7)), 0
    for i in range(1, 7):
        e = rng.random((10, 14)) * 0.05
        fl = F.MotionField(16, 14, 10, np.zeros((10, 14, 2), np.int64), e, np.ones((10, 14), bool))
        d, st = FS.decide(st, fl, i, 0.1, None, "mean")
        kind, ref, trig, acc, fsk = O.decide(acc, fsk, 32, e, 16, i, 0.1, None, "mean")
        assert d.kind.value == kind and d.trigger_statistic == trig
        np.testing.assert_array_equal(st.accumulated, acc)
