"""Device-time split of one C2 bench step: the three captured graphs (pack+reset | ME | refine+AEM+chain),
bracketed by CUDA events, L2 flushed before each step as in bench.py."""
import sys, statistics
sys.path.insert(0, '.'); sys.path.insert(0, 'tools')
import numpy as np, torch
import bench
import _variant
_variant.use_variant_from_env()
from paper_2508_05990_b200.engine import ClipEngine
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
c = bench.CONFIGS[name]
clip, labels = bench.make_clip(name)
pcfg = bench.pipeline_config(name)
eng = ClipEngine(pcfg, c[1], c[0], c[2], 1, clip.dtype, True)
eng.load_frames(clip[None])
for t in range(c[2]):
    eng.key_labels[0, t].copy_(torch.from_numpy(labels[t].classes.copy()))
eng.capture()
flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.int32, device="cuda")
res = []
for k in range(13):
    flush.fill_(1)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    ev[0].record()
    for i, g in enumerate(eng.graph):
        g.replay()
        ev[i + 1].record()
    torch.cuda.synchronize()
    if k >= 3:
        res.append([ev[i].elapsed_time(ev[i + 1]) * 1e3 for i in range(3)])
m = [statistics.median(r[i] for r in res) for i in range(3)]
print(f"pre {m[0]:.1f} us | ME {m[1]:.1f} us | post {m[2]:.1f} us | total {sum(m):.1f} us")

# eager split of the post-ME work (same stream, events between the C-ABI calls)
parts = [("refine", lambda: eng._refine(0, eng.n_pairs)), ("decide", lambda: eng._decide(1, eng.T)),
         ("chain", eng.predict), ("reset", eng._reset_state), ("pack", eng._pack)]
acc = {n: [] for n, _ in parts}
for k in range(13):
    flush.fill_(1)
    for g in eng.graph:
        g.replay()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(parts) + 1)]
    ev[0].record()
    for i, (n, f) in enumerate(parts):
        f()
        ev[i + 1].record()
    torch.cuda.synchronize()
    if k >= 3:
        for i, (n, _) in enumerate(parts):
            acc[n].append(ev[i].elapsed_time(ev[i + 1]) * 1e3)
print(" | ".join(f"{n} {statistics.median(v):.1f} us" for n, v in acc.items()))
