"""Host-side cost of ClipSession.run on a bench config: wall time per method (Python + launch
overhead; _finish_chunk's wait for the decisions measured separately)."""
import sys, time, json
from collections import defaultdict
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import bench
from paper_2508_05990_b200 import pipeline
from paper_2508_05990_b200.pipeline import ClipSession
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
chunks = int(sys.argv[2]) if len(sys.argv) > 2 else 10
c = bench.CONFIGS[name]
pcfg = bench.pipeline_config(name)
clip, labels = bench.make_clip(name)
raw = torch.from_numpy(clip).pin_memory()
lab = torch.from_numpy(np.stack([l.classes for l in labels])).pin_memory()
acc = defaultdict(float)
def wrap(cls, meth):
    f = getattr(cls, meth)
    def g(*a, **k):
        t0 = time.perf_counter(); r = f(*a, **k); acc[meth] += time.perf_counter() - t0; return r
    setattr(cls, meth, g)
for m in ("_motion_chunk", "_decisions_out", "_finish_chunk"):
    wrap(ClipSession, m)
orig_sync = torch.cuda.Event.synchronize
def sync(self):
    t0 = time.perf_counter(); orig_sync(self); acc["event_wait"] += time.perf_counter() - t0
torch.cuda.Event.synchronize = sync
sess = ClipSession(pcfg, c[1], c[0], c[2], clip.dtype, True, chunks=chunks)
for _ in range(3):
    sess.run(raw, lab)
torch.cuda.synchronize()
acc.clear()
n = 10
t0 = time.perf_counter()
for _ in range(n):
    sess.run(raw, lab)
torch.cuda.synchronize()
tot = (time.perf_counter() - t0) / n
print(json.dumps({"config": name, "chunks": chunks, "ms_per_run": round(1e3 * tot, 3),
                  **{k: round(1e3 * v / n, 3) for k, v in acc.items()}}))
