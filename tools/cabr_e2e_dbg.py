"""Compare the weighted label chain across execution paths on a bench config:
direct engine calls, captured graph replay, ClipSession (chunks 10 and 1)."""
import sys
from dataclasses import replace
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2508_05990_b200 import cabr  # noqa: E402
from paper_2508_05990_b200.engine import ClipEngine  # noqa: E402
from paper_2508_05990_b200.pipeline import ClipSession  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5cabr"
W, H, T = bench.CONFIGS[name][:3]
pcfg = bench.pipeline_config(name)
clip, labels = bench.make_clip(name)
keys = np.stack([l.classes for l in labels])
w = cabr.random_weights(bench.CABR_CLASSES.get(name, 19), seed=0)


def engine(capture):
    eng = ClipEngine(pcfg, H, W, T, 1, clip.dtype, True)
    eng.load_frames(clip)
    eng.key_labels[0].copy_(torch.from_numpy(keys))
    eng.set_cabr(w)
    if capture:
        eng.capture()
        for _ in range(3):
            eng.replay()
    else:
        eng.step()
    torch.cuda.synchronize()
    return eng.labels[0].cpu().numpy(), eng.kind[0].cpu().numpy()


A, kinds = engine(False)
B, _ = engine(True)
outs = {"graph": B}
for ch in (10, 1):
    sess = ClipSession(pcfg, H, W, T, clip.dtype, True, chunks=ch, weights=w)
    for _ in range(2):
        got, _, _, _ = sess.run(torch.from_numpy(clip).pin_memory(), torch.from_numpy(keys).pin_memory())
    outs[f"session{ch}"] = np.stack(got)
for k, v in outs.items():
    bad = [t for t in range(T) if kinds[t] != 0 and not np.array_equal(v[t], A[t])]
    print(k, "differing predicted frames:", bad[:10], "pixels:", [int((v[t] != A[t]).sum()) for t in bad[:5]])
