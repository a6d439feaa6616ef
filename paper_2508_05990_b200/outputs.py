"""Run-output writers: the files the reference's CLI
produces around the hot path, with identical names, formats and content.

* ``write_estimate_outputs``  motion-field JSON with all ``levels`` plus the
  refined final field, and the energy PGM (cli.py:84-98);
* ``run_report``              the ``report.json`` dictionary of ``bayermc run``
  (cli.py:146-176) -- per-frame mIoU comes from the GPU confusion kernel
  (``metrics.miou_clip``: all frames in one launch);
* ``write_run_outputs``       ``labels/<name>.png``, ``decisions.jsonl``,
  ``ledger.json``, ``report.json``, ``report.txt`` (cli.py:108-123).

The argparse CLI itself is out of scope (SURVEY.md §8 tier); these functions are
what it calls, so a maintainer can bind them under the same subcommands.
"""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np

from . import frame_io, metrics
from .fme import MotionField, save_motion_field


def energy_image(field: MotionField) -> frame_io.Frame:
    """Energy grid as an 8-bit luma frame: clip(rint(E*255), 0, 255) (cli.py:93-97)."""
    energy = np.clip(np.rint(np.asarray(field.energy) * 255.0), 0, 255).astype(np.uint8)
    return frame_io.Frame(width=field.grid_w, height=field.grid_h, data=energy)


def write_estimate_outputs(fields, refined: MotionField, out_path, energy_path=None) -> Path:
    """``bayermc estimate`` outputs: JSON of the non-final levels + the refined final
    field, and ``<stem>_energy.pgm`` (or ``energy_path``).  Returns the energy path."""
    out_path = Path(out_path)
    save_motion_field(list(fields[:-1]) + [refined], out_path)
    energy_path = Path(energy_path) if energy_path else out_path.with_name(out_path.stem + "_energy.pgm")
    frame_io.save_frame(energy_image(refined), energy_path)
    return energy_path


def run_report(result, backbone_gflops: float, truth=None, num_classes: int | None = None) -> dict:
    """``report.json`` of ``bayermc run`` (cli.py:146-176).  ``truth`` is an optional
    list (one per frame) of ground-truth LabelMaps or None."""
    frames = len(result.labels)
    report = {
        "frames": frames,
        "keyframes": result.keyframes,
        "scale": result.scale,
        "components": result.ledger.as_dict(),
        "backbone_gflops_per_keyframe": backbone_gflops,
        "average_gflops_per_frame": metrics.ledger_report(result.ledger, backbone_gflops, frames,
                                                          result.keyframes),
    }
    if truth is not None:
        have = [i for i, t in enumerate(truth) if t is not None]
        per_frame = [None] * frames
        if have:
            # cli.py:161-166 scores each frame with miou(labels, truth): num_classes is the max of both maps'
            groups = {}
            for i in have:
                nc = num_classes or max(result.labels[i].num_classes, truth[i].num_classes)
                groups.setdefault(nc, []).append(i)
            for nc, idx in groups.items():
                scores = metrics.miou_clip(np.stack([result.labels[i].classes for i in idx]),
                                           np.stack([truth[i].classes for i in idx]), nc)
                for i, s in zip(idx, scores):
                    per_frame[i] = s
        report["miou_per_frame"] = per_frame
        nonkey = [per_frame[i] for i in have if result.decisions[i].kind.value != "key"]
        if nonkey:
            report["miou_mean_nonkey"] = sum(nonkey) / len(nonkey)
    return report


def write_run_outputs(result, names, out_dir, report: dict) -> None:
    """The ``bayermc run`` output directory (cli.py:108-123)."""
    out_dir = Path(out_dir)
    labels_dir = out_dir / "labels"
    labels_dir.mkdir(parents=True, exist_ok=True)
    for name, labels in zip(names, result.labels):
        frame_io.save_labels(labels, labels_dir / (name + ".png"))
    with open(out_dir / "decisions.jsonl", "w", encoding="utf-8") as fh:
        for decision in result.decisions:
            fh.write(json.dumps(decision.to_json_dict()) + "\n")
    (out_dir / "ledger.json").write_text(result.ledger.to_json() + "\n", encoding="utf-8")
    (out_dir / "report.json").write_text(json.dumps(report, indent=1) + "\n", encoding="utf-8")
    (out_dir / "report.txt").write_text(result.ledger.table() + "\n", encoding="utf-8")
