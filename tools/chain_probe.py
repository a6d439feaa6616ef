"""Label-chain timing split: C2 clip, fixed GOP, ring vote on/off, various GOP lengths (eager C-ABI calls, events)."""
import sys, statistics
sys.path.insert(0, '.'); sys.path.insert(0, 'tools')
import numpy as np, torch
import bench, _variant
_variant.use_variant_from_env()
from paper_2508_05990_b200.config import PipelineConfig
from paper_2508_05990_b200.engine import ClipEngine
clip, labels = bench.make_clip("c2")
base = bench.pipeline_config("c2")
import dataclasses
for ring in (False, True):
    for gop in (2, 6, 30):
        pcfg = dataclasses.replace(base, max_gop=gop, aem_threshold=float("inf"), refine_enabled=ring)
        eng = ClipEngine(pcfg, 1080, 1920, 30, 1, clip.dtype, True)
        eng.load_frames(clip[None])
        eng.key_labels[0].copy_(torch.from_numpy(np.stack([l.classes for l in labels])))
        eng.motion(); eng.predict(); torch.cuda.synchronize()
        ts = []
        for k in range(12):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); eng.predict(); e1.record(); torch.cuda.synchronize()
            if k >= 2: ts.append(e0.elapsed_time(e1) * 1e3)
        pred = int((eng.kind[0] != 0).sum())
        print(f"ring={ring} gop={gop} predicted={pred} chain {statistics.median(ts):.1f} us "
              f"({(statistics.median(ts)) / max(pred, 1):.1f} us/predicted frame)", flush=True)
