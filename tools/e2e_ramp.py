"""e2e of ClipSession.run (native session) over (chunks, lag, ramp) on a bench config."""
import sys, time, json
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import bench
from paper_2508_05990_b200.pipeline import ClipSession
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
c = bench.CONFIGS[name]
pcfg = bench.pipeline_config(name)
clip, labels = bench.make_clip(name)
raw = torch.from_numpy(clip).pin_memory()
lab = torch.from_numpy(np.stack([l.classes for l in labels])).pin_memory()
for chunks, lag, ramp in [(5, 2, 1.0), (5, 1, 1.0), (5, 3, 1.0), (6, 2, 1.5), (8, 2, 1.5), (8, 3, 1.5), (10, 3, 1.5),
                          (6, 2, 2.0), (8, 3, 2.0), (4, 2, 1.5), (4, 1, 1.5), (3, 1, 1.5)]:
    sess = ClipSession(pcfg, c[1], c[0], c[2], clip.dtype, True, chunks=chunks, lag=lag, ramp=ramp)
    for _ in range(3):
        sess.run(raw, lab)
    ts = []
    for _ in range(20):
        torch.cuda.synchronize(); t0 = time.perf_counter(); sess.run(raw, lab); ts.append(1e3 * (time.perf_counter() - t0))
    print(json.dumps({"config": name, "chunks": chunks, "lag": lag, "ramp": ramp, "bounds": [a for a, _ in sess.chunks],
                      "ms_med": round(float(np.median(ts)), 3)}), flush=True)
