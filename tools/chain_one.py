"""One C2 fixed-GOP (max_gop=6) label chain with ring vote, for ncu."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch, dataclasses
import bench
from paper_2508_05990_b200.engine import ClipEngine
clip, labels = bench.make_clip("c2")
pcfg = dataclasses.replace(bench.pipeline_config("c2"), max_gop=6, aem_threshold=float("inf"), refine_enabled=True)
eng = ClipEngine(pcfg, 1080, 1920, 30, 1, clip.dtype, True)
eng.load_frames(clip[None])
eng.key_labels[0].copy_(torch.from_numpy(np.stack([l.classes for l in labels])))
eng.motion(); torch.cuda.synchronize()
m = eng.levels[-1].matched[:eng.n_pairs]
print("flagged blocks per pair:", (m == 0).sum().item() / eng.n_pairs, flush=True)
for _ in range(3):
    eng.predict()
torch.cuda.synchronize()
