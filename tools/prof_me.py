"""Drive the dominant kernel for ncu: C2 clip, one ME launch over all 29 pairs (after warm-up)."""
import sys, ctypes
sys.path.insert(0, '.')
import torch
import bench
from paper_2508_05990_b200 import _native as N
from paper_2508_05990_b200.engine import ClipEngine
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
c = bench.CONFIGS[name]
clip, labels = bench.make_clip(name)
eng = ClipEngine(bench.pipeline_config(name), c[1], c[0], c[2], 1, clip.dtype, True)
eng.load_frames(clip)
eng.step()
torch.cuda.synchronize()
arr = eng._level_slice(0, eng.n_pairs)
for _ in range(reps):
    N.check(N.load().bmc_estimate_motion(N.ptr(eng.planes), eng.S * eng.T, ctypes.byref(eng.params), eng.n_pairs,
                                         N.ptr(eng.cur_index), N.ptr(eng.ref_index), arr, N.stream_handle()))
torch.cuda.synchronize()
print("done")
