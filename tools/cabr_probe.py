"""Time the weighted label chain (bmc_cabr_chain) on a bench config: flagged blocks,
chain ms, executed fp32 FLOP rate.  usage: python tools/cabr_probe.py c5 [classes] [reps]"""
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2508_05990_b200 import cabr  # noqa: E402
from paper_2508_05990_b200.engine import ClipEngine  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
C = int(sys.argv[2]) if len(sys.argv) > 2 else 19
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
W, H, T = bench.CONFIGS[name][:3]
pcfg = bench.pipeline_config(name)
from dataclasses import replace  # noqa: E402
pcfg = replace(pcfg, refine_enabled=True)
clip, labels = bench.make_clip(name)
eng = ClipEngine(pcfg, H, W, T, 1, clip.dtype, True)
eng.load_frames(clip)
eng.motion()
for t in range(T):
    eng.key_labels[0, t].copy_(torch.from_numpy(labels[t].classes % C))
w = cabr.random_weights(C, seed=0)
eng.set_cabr(w)
eng.predict()
torch.cuda.synchronize()
kinds = eng.kind.cpu().numpy()[0]
m = eng.levels[-1].matched[:eng.n_pairs].cpu().numpy()
flag = sum(int((m[t - 1] == 0).sum()) for t in range(1, T) if kinds[t] != 0)
K = eng.b_final * eng.scale
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ms = []
for _ in range(reps):
    ev[0].record()
    eng.predict()
    ev[1].record()
    torch.cuda.synchronize()
    ms.append(ev[0].elapsed_time(ev[1]))
ms_med = float(np.median(ms))
ex = cabr.executed_flops(K, C) * flag
ref = cabr.count_cabr_flops(K, C, flag)
print(json.dumps({"config": name, "K": K, "classes": C, "predicted": int((kinds != 0).sum()), "flagged_blocks": flag,
                  "chain_ms": ms_med, "executed_gflop": ex / 1e9, "reference_gflop": ref / 1e9,
                  "executed_tflops": ex / ms_med / 1e9, "reference_equiv_tflops": ref / ms_med / 1e9}))
