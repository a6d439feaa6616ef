"""Time ClipSession.run (host buffers) for the C2 clip with several chunk counts / label forms."""
import sys, time, statistics
sys.path.insert(0, '.')
import numpy as np, torch
import bench
from paper_2508_05990_b200.pipeline import ClipSession
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
c = bench.CONFIGS[name]
clip, labels = bench.make_clip(name)
pcfg = bench.pipeline_config(name)
raw = torch.from_numpy(clip).pin_memory()
lab_t = torch.from_numpy(np.stack([l.classes for l in labels])).pin_memory()
lab_d = {i: l for i, l in enumerate(labels)}
for chunks in (1, 2, 3, 6):
    sess = ClipSession(pcfg, c[1], c[0], c[2], clip.dtype, True, chunks=chunks)
    for form, key in (("tensor", lab_t), ("dict", lab_d)):
        for _ in range(2):
            sess.run(raw, key)
        ts = []
        for _ in range(5):
            torch.cuda.synchronize(); t0 = time.perf_counter()
            sess.run(raw, key)
            ts.append(1e3 * (time.perf_counter() - t0))
        print(f"chunks={chunks} {form}: median {statistics.median(ts):.2f} ms  min {min(ts):.2f}", flush=True)
