"""Drive the round-2 kernels once each for compute-sanitizer: the SEA screening and
cooperative replays (C1 unit-step stage; a 64-pixel-block C5 clip), the native session
executor, and the CaBR-Net chain / blocks / refine (K = 16)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_2508_05990_b200 import cabr, pipeline, synth
from paper_2508_05990_b200.config import PipelineConfig
from paper_2508_05990_b200.fme import FmeConfig, SearchStage, get_preset
from paper_2508_05990_b200.frame_io import Frame, FrameKind

# SEA (unit-step +-8 search over 16x16 blocks) + selection
clip = synth.bayer_pan_clip(256, 256, 4, (2, 2), seed=3)
labels = synth.block_labels(256, 256, 4)
f1 = FmeConfig(stages=(SearchStage(8, 1), SearchStage(0, 1), SearchStage(0, 1)), block_sizes=(16,))
frames = [Frame(256, 256, c, FrameKind.BAYER_RGGB) for c in clip]
pipeline.run_sequence(frames, {i: l for i, l in enumerate(labels)}, PipelineConfig(fme=f1, refine_enabled=False))
# native session (chunked) on the same clip
sess = pipeline.ClipSession(PipelineConfig(fme=f1, refine_enabled=False), 256, 256, 4, np.uint8, True, chunks=2)
sess.run(torch.from_numpy(clip).pin_memory(), torch.from_numpy(np.stack([l.classes for l in labels])).pin_memory())
# large blocks (64 -> 32): cooperative replays
c5 = synth.bayer_pan_clip(320, 256, 3, (6, -4), seed=8, square=48, square_velocity=(7, 3))
fr5 = [Frame(320, 256, c, FrameKind.BAYER_RGGB) for c in c5]
lab5 = synth.block_labels(320, 256, 3, num_classes=5, seed=1)
pipeline.run_sequence(fr5, {i: l for i, l in enumerate(lab5)}, PipelineConfig(fme=get_preset("standard"),
                                                                               refine_enabled=False))
# CaBR-Net: weighted chain (K = 16), blocks API, refine_blocks
f2 = FmeConfig(stages=(SearchStage(4, 2), SearchStage(1, 1), SearchStage(1, 1)), block_sizes=(16, 8))
c2 = synth.bayer_pan_clip(160, 128, 3, (2, -3), seed=12, square=40, square_velocity=(6, 2))
fr2 = [Frame(160, 128, c, FrameKind.BAYER_RGGB) for c in c2]
lab2 = synth.block_labels(160, 128, 3, num_classes=4, seed=9)
w = cabr.random_weights(4, seed=14)
pipeline.run_sequence(fr2, {i: l for i, l in enumerate(lab2)},
                      PipelineConfig(fme=f2, max_gop=3, aem_threshold=float("inf")), weights=w)
cabr.cabr_forward_blocks(fr2[0], lab2[0], [(0, 0), (150, 120)], 32, w)
cabr.refine_blocks(fr2[0], lab2[0], [(0, 0), (16, 16), (150, 120)], 16, w)
cabr.refine_blocks(fr2[0], lab2[0], [(0, 0), (16, 16), (150, 120)], 16, None)
torch.cuda.synchronize()
print("ok")
