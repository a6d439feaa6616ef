import sys, time, statistics
sys.path.insert(0, '.')
import numpy as np, torch
import bench
from paper_2508_05990_b200.pipeline import ClipSession
from paper_2508_05990_b200.engine import ClipEngine
c = bench.CONFIGS["c2"]; clip, labels = bench.make_clip("c2"); pcfg = bench.pipeline_config("c2")
raw = torch.from_numpy(clip).pin_memory()
lab_t = torch.from_numpy(np.stack([l.classes for l in labels])).pin_memory()
def t(sess, tag, flush=None):
    for _ in range(2): sess.run(raw, lab_t)
    ts=[]
    for _ in range(5):
        if flush is not None: flush.fill_(1)
        torch.cuda.synchronize(); t0=time.perf_counter(); sess.run(raw, lab_t); ts.append(1e3*(time.perf_counter()-t0))
    print(tag, f"{statistics.median(ts):.2f}", flush=True)
sess = ClipSession(pcfg, c[1], c[0], c[2], clip.dtype, True)
t(sess, "plain")
flush = torch.empty(512*1024*1024//4, dtype=torch.int32, device="cuda")
t(sess, "flush", flush)
eng = ClipEngine(pcfg, c[1], c[0], c[2], 1, clip.dtype, True); eng.load_frames(clip); eng.capture(); eng.replay(); torch.cuda.synchronize()
t(sess, "after-engine-capture")
t(sess, "after-engine-capture+flush", flush)
sess2 = ClipSession(pcfg, c[1], c[0], c[2], clip.dtype, True)
t(sess2, "new-session-after-capture")
