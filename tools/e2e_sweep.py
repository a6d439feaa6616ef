"""ClipSession e2e timing sweep over (chunks, lag) for a bench config (C2 / C2gop)."""
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
for chunks in (5, 6, 8, 10, 15):
    for lag in (1, 2, 3, 4):
        sess = ClipSession(pcfg, c[1], c[0], c[2], clip.dtype, True, chunks=chunks, lag=lag)
        for _ in range(3):
            sess.run(raw, lab)
        ts = []
        for _ in range(15):
            torch.cuda.synchronize(); t0 = time.perf_counter(); sess.run(raw, lab); ts.append(1e3 * (time.perf_counter() - t0))
        print(json.dumps({"config": name, "chunks": chunks, "lag": lag, "ms_med": round(float(np.median(ts)), 3),
                          "ms_min": round(min(ts), 3), "h2d": sess.h2d_bytes, "d2h": sess.d2h_bytes}), flush=True)
