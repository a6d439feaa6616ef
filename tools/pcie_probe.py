"""PCIe bandwidth and e2e chunking probe for the C2 host-buffer path (ClipSession.run).

Prints pinned H2D / D2H bandwidth (alone and concurrent) and the e2e time of
ClipSession.run for several chunkings, so the streamed schedule can be compared
with its copy-bound floor.
"""
import sys, time, statistics
sys.path.insert(0, '.')
import numpy as np, torch
import bench
from paper_2508_05990_b200.pipeline import ClipSession


def ev_time(fn, reps=5):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(1e3 * (time.perf_counter() - t0))
    return statistics.median(ts)


MB = 1 << 20
h = torch.empty(124 * MB, dtype=torch.uint8).pin_memory()
d = torch.empty(124 * MB, dtype=torch.uint8, device="cuda")
ho = torch.empty(62 * MB, dtype=torch.uint8).pin_memory()
do = torch.empty(62 * MB, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
t = ev_time(lambda: d.copy_(h, non_blocking=True))
print(f"H2D 124MB: {t:.3f} ms = {124 * MB / t / 1e6:.1f} GB/s")
t = ev_time(lambda: ho.copy_(do, non_blocking=True))
print(f"D2H 62MB: {t:.3f} ms = {62 * MB / t / 1e6:.1f} GB/s")


def both():
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        ho.copy_(do, non_blocking=True)


t = ev_time(both)
print(f"H2D 124MB || D2H 62MB: {t:.3f} ms")

c = bench.CONFIGS["c2"]
clip, labels = bench.make_clip("c2")
pcfg = bench.pipeline_config("c2")
raw = torch.from_numpy(clip).pin_memory()
lab = torch.from_numpy(np.stack([l.classes for l in labels])).pin_memory()
for k in (3, 6, 10, 15, 30):
    sess = ClipSession(pcfg, c[1], c[0], c[2], clip.dtype, True, chunks=k)
    for _ in range(2):
        sess.run(raw, lab)
    t = ev_time(lambda: sess.run(raw, lab), 7)
    print(f"ClipSession chunks={k}: {t:.3f} ms/clip = {29 / t * 1e3:.0f} frames/s")
