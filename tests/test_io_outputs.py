"""File ingest, mIoU and run-output writers against files and values the REFERENCE
itself wrote (tests/golden/make_golden_io.py -> tests/golden/io/)."""

import json
from pathlib import Path

import numpy as np
import pytest

IO = Path(__file__).resolve().parent / "golden" / "io"


def _npz():
    return dict(np.load(IO / "io.npz", allow_pickle=False))


# ----------------------------------------------------------------------------- CPU
def test_pgm_header_errors_match_reference(tmp_path):
    from paper_2508_05990_b200 import ingest
    with pytest.raises(ValueError, match="not a binary PGM"):
        ingest.parse_pgm_header(b"P2\n1 1\n255\n0", "x.pgm")
    with pytest.raises(ValueError, match="truncated PGM header"):
        ingest.parse_pgm_header(b"P5\n1 1", "x.pgm")
    with pytest.raises(ValueError, match="unsupported PGM maxval 70000"):
        ingest.parse_pgm_header(b"P5\n1 1\n70000\n\0\0", "x.pgm")
    assert ingest.parse_pgm_header((IO / "comment.pgm").read_bytes(), "c")[:3] == (10, 6, 4095)


def test_u8_pgm_png_and_labels_load_like_reference():
    from paper_2508_05990_b200 import frame_io
    d = _npz()
    np.testing.assert_array_equal(frame_io.load_frame(IO / "u8.pgm").data, d["u8_pgm"])
    np.testing.assert_array_equal(frame_io.load_labels(IO / "labels.png").classes, d["labels_png"])
    assert frame_io.load_labels(IO / "labels.png").num_classes == int(d["labels_png"].max()) + 1
    with pytest.raises(ValueError, match="cannot infer format"):
        frame_io.load_frame(IO / "c1.toml")


def test_mipi_host_encoder_layout():
    from paper_2508_05990_b200 import ingest
    px = np.array([[0x3FF, 0x001, 0x2AA, 0x155]], np.uint16)
    b = ingest.pack_mipi(px, 10)
    assert b.tolist() == [[0xFF, 0x00, 0xAA, 0x55, 0b01_10_01_11]]
    px12 = np.array([[0xABC, 0x123]], np.uint16)
    assert ingest.pack_mipi(px12, 12).tolist() == [[0xAB, 0x12, 0x3C]]


def test_energy_image_rounding():
    from paper_2508_05990_b200 import outputs
    from paper_2508_05990_b200.fme import MotionField
    f = MotionField(16, 3, 1, np.zeros((1, 3, 2), np.int64), np.array([[0.0, 0.5 / 255, 2.0]]),
                    np.ones((1, 3), bool))
    assert outputs.energy_image(f).data.tolist() == [[0, 0, 255]]


def test_miou_oracle_matches_reference_values():
    from oracle import bayermc_oracle as O
    d = _npz()
    for k in range(6):
        ign = int(d[f"miou{k}_ignore"])
        v = O.miou(d[f"miou{k}_pred"], d[f"miou{k}_truth"], int(d[f"miou{k}_nc"]), None if ign < 0 else ign)
        assert v == float(d[f"miou{k}_value"]), k


# ----------------------------------------------------------------------------- GPU
@pytest.mark.gpu
def test_pgm_png_loads_match_reference(cuda):
    from paper_2508_05990_b200 import frame_io
    d = _npz()
    for name in ("u16.pgm", "u8.pgm", "comment.pgm", "u16.png"):
        got = frame_io.load_frame(IO / name).data
        want = d[name.replace(".", "_")]
        assert got.dtype == want.dtype
        np.testing.assert_array_equal(got, want)


@pytest.mark.gpu
def test_save_frame_bytes_match_reference(cuda, tmp_path):
    from paper_2508_05990_b200 import frame_io
    d = _npz()
    frame_io.save_frame(frame_io.Frame(64, 48, d["u16_pgm"]), tmp_path / "a.pgm")
    assert (tmp_path / "a.pgm").read_bytes() == (IO / "u16.pgm").read_bytes()
    frame_io.save_frame(frame_io.Frame(40, 30, d["u8_pgm"]), tmp_path / "b.pgm")
    assert (tmp_path / "b.pgm").read_bytes() == (IO / "u8.pgm").read_bytes()


@pytest.mark.gpu
@pytest.mark.parametrize("bits", [10, 12])
def test_mipi_raw_decode_on_gpu(cuda, tmp_path, bits):
    from paper_2508_05990_b200 import frame_io, ingest
    rng = np.random.default_rng(bits)
    frames = rng.integers(0, 1 << bits, (3, 36, 72)).astype(np.uint16)
    packed = ingest.pack_mipi(frames, bits)
    out = ingest.decode(packed, 72, 36, f"raw{bits}", frames=3).cpu().numpy()
    np.testing.assert_array_equal(out, frames)
    # padded line stride (CSI-2 line alignment) and left alignment to 16 bits
    stride = packed.shape[-1] + 27
    padded = np.zeros((3, 36, stride), np.uint8)
    padded[..., :packed.shape[-1]] = packed
    out = ingest.decode(padded, 72, 36, f"raw{bits}", frames=3, row_bytes=stride, shift=16 - bits)
    np.testing.assert_array_equal(out.cpu().numpy(), frames << (16 - bits))
    (tmp_path / "f.raw").write_bytes(packed[1].tobytes())
    fr = frame_io.load_raw_frame(tmp_path / "f.raw", 72, 36, bits)
    np.testing.assert_array_equal(fr.data, frames[1])
    assert fr.kind.is_bayer


@pytest.mark.gpu
def test_be16_decode_odd_width_and_unaligned(cuda):
    from paper_2508_05990_b200 import ingest
    rng = np.random.default_rng(5)
    a = rng.integers(0, 65536, (2, 7, 13)).astype(np.uint16)
    payload = np.concatenate([np.zeros(3, np.uint8), np.frombuffer(a.astype(">u2").tobytes(), np.uint8)])
    t = cuda.from_numpy(payload).cuda()[3:]  # deliberately misaligned source
    np.testing.assert_array_equal(ingest.decode(t, 13, 7, "be16", frames=2).cpu().numpy(), a)


@pytest.mark.gpu
def test_pgm_clip_reader(cuda):
    from paper_2508_05990_b200 import frame_io, ingest
    paths = sorted((IO / "frames").glob("*.pgm"))
    rd = ingest.PgmClipReader()
    clip = rd.read(paths).cpu().numpy()
    np.testing.assert_array_equal(clip, np.stack([frame_io.load_frame(p).data for p in paths]))
    clip2 = rd.read([IO / "u16.pgm", IO / "u16.pgm"]).cpu().numpy()
    np.testing.assert_array_equal(clip2[1], _npz()["u16_pgm"])


@pytest.mark.gpu
def test_miou_gpu_matches_reference_values(cuda):
    from paper_2508_05990_b200 import metrics
    from paper_2508_05990_b200.frame_io import LabelMap
    d = _npz()
    for k in range(6):
        t, p, nc = d[f"miou{k}_truth"], d[f"miou{k}_pred"], int(d[f"miou{k}_nc"])
        ign = int(d[f"miou{k}_ignore"])
        h, w = t.shape
        got = metrics.miou(LabelMap(w, h, p, nc), LabelMap(w, h, t, nc), ignore_class=None if ign < 0 else ign)
        assert got == float(d[f"miou{k}_value"]), k
    with pytest.raises(ValueError, match="dimension mismatch"):
        metrics.miou(LabelMap(2, 1, np.zeros((1, 2), np.uint8), 2), LabelMap(1, 2, np.zeros((2, 1), np.uint8), 2))
    # a large batched call: 4K maps, 19 classes, clip of 6
    rng = np.random.default_rng(3)
    truth = rng.integers(0, 19, (6, 2160, 3840)).astype(np.uint8)
    pred = np.where(rng.random(truth.shape) < 0.8, truth, 0).astype(np.uint8)
    from oracle import bayermc_oracle as O
    got = metrics.miou_clip(pred, truth, 19)
    assert got == [O.miou(pred[i], truth[i], 19) for i in range(6)]


@pytest.mark.gpu
def test_run_outputs_match_reference_cli(cuda, tmp_path):
    """The `bayermc run` flow on PGM/PNG files: every output file equals the one the
    reference's CLI wrote (decisions.jsonl, ledger.json, report.json, report.txt, label PNGs)."""
    from paper_2508_05990_b200 import frame_io, outputs, pipeline
    from paper_2508_05990_b200.config import load_pipeline_config
    import dataclasses
    cfg = dataclasses.replace(load_pipeline_config(IO / "c1.toml"), max_gop=3)
    files = sorted((IO / "frames").glob("*.pgm"))
    frames = [frame_io.load_frame(p, kind=frame_io.FrameKind.BAYER_RGGB) for p in files]
    names = [p.stem for p in files]
    res = pipeline.run_sequence(frames, lambda i: frame_io.load_labels(IO / "keys" / (names[i] + ".png"),
                                                                      num_classes=19), cfg)
    truth = [frame_io.load_labels(IO / "truth" / (n + ".png"), num_classes=19) for n in names]
    report = outputs.run_report(res, cfg.backbone_gflops, truth)
    outputs.write_run_outputs(res, names, tmp_path, report)
    for name in ("decisions.jsonl", "ledger.json", "report.json", "report.txt"):
        assert (tmp_path / name).read_text() == (IO / "run" / name).read_text(), name
    for n in names:
        got = frame_io.load_labels(tmp_path / "labels" / (n + ".png")).classes
        np.testing.assert_array_equal(got, frame_io.load_labels(IO / "run" / "labels" / (n + ".png")).classes)
    assert json.loads((tmp_path / "report.json").read_text())["keyframes"] == 4


@pytest.mark.gpu
def test_estimate_outputs_match_reference_cli(cuda, tmp_path):
    from paper_2508_05990_b200 import fme, frame_io, mv_refine, outputs
    from paper_2508_05990_b200.config import load_pipeline_config
    cfg = load_pipeline_config(IO / "c1.toml")
    kind = frame_io.FrameKind.BAYER_RGGB
    cur = frame_io.load_frame(IO / "frames" / "f001.pgm", kind=kind)
    ref = frame_io.load_frame(IO / "frames" / "f000.pgm", kind=kind)
    fields = fme.estimate_motion(cur, ref, cfg.fme)
    refined = mv_refine.refine_mvs(fields[-1], cfg.deviation_threshold, cur=cur, ref=ref, config=cfg.fme)
    epath = outputs.write_estimate_outputs(fields, refined, tmp_path / "field.json")
    assert epath.name == "field_energy.pgm"
    assert (tmp_path / "field.json").read_text() == (IO / "estimate" / "field.json").read_text()
    assert epath.read_bytes() == (IO / "estimate" / "field_energy.pgm").read_bytes()
