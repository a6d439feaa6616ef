"""Time the ME launch of a config (CUDA events, L2 flushed between reps); prints one JSON line."""
import sys, ctypes, json, os, statistics
sys.path.insert(0, '.'); sys.path.insert(0, 'tools')
import torch
import bench
import _variant
_variant.use_variant_from_env()
from paper_2508_05990_b200 import _native as N
from paper_2508_05990_b200.engine import ClipEngine
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
c = bench.CONFIGS[name]
clip, labels = bench.make_clip(name)
pcfg = bench.pipeline_config(name)
eng = ClipEngine(pcfg, c[1], c[0], c[2], 1, clip.dtype, True)
eng.load_frames(clip)
eng.step()
torch.cuda.synchronize()
arr = eng._level_slice(0, eng.n_pairs)
flush = torch.empty(128 * 1024 * 1024, dtype=torch.int32, device="cuda")
ts = []
for k in range(reps + 2):
    flush.fill_(k)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    N.check(N.load().bmc_estimate_motion(N.ptr(eng.planes), eng.S * eng.T, ctypes.byref(eng.params), eng.n_pairs,
                                         N.ptr(eng.cur_index), N.ptr(eng.ref_index), arr, N.stream_handle()))
    e1.record(); e1.synchronize()
    if k >= 2: ts.append(e0.elapsed_time(e1))
evals = [int(lv.evals[:eng.n_pairs].sum().item()) for lv in eng.levels]
samples = sum(e * 4 * b * b for e, b in zip(evals, pcfg.fme.block_sizes))
ms = statistics.median(ts)
bpp = clip.dtype.itemsize
peak = (256 if bpp == 1 else 64) * 148 * 1965e6
print(json.dumps({"variant": os.environ.get("VARIANT", "?"), "cfg": name, "ty_max": os.environ.get("BMC_TY_MAX", "12"),
                  "me_ms": round(ms, 4), "frac": round(samples / (ms / 1e3) / peak, 4), "evals": evals}))
