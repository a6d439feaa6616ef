"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck):
every product kernel once on C1-sized inputs.

    compute-sanitizer --tool racecheck python tools/sanitize_c1.py

* fme_stage_kernel (TMA + mbarrier staging): C1 full +-8 search, b16
* fme_small_kernel: 8x8 Bayer blocks, 3-stage schedule
* refine / decide / pack kernels and the cooperative label chain with the ring
  vote (grid barrier): run_sequence with refine_enabled on C1
"""

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402

from paper_2508_05990_b200 import fme, pipeline, synth  # noqa: E402
from paper_2508_05990_b200.config import PipelineConfig  # noqa: E402
from paper_2508_05990_b200.fme import FmeConfig, SearchStage  # noqa: E402


def main():
    clip = synth.bayer_pan_clip(256, 256, 4, (2, 2), seed=3, square=64, square_velocity=(5, -3))
    fr = synth.frames_of(clip)
    c1 = FmeConfig(stages=(SearchStage(8, 1), SearchStage(0, 1), SearchStage(0, 1)), block_sizes=(16,))
    f = fme.estimate_motion(fr[1], fr[0], c1)
    small = FmeConfig(stages=(SearchStage(4, 8), SearchStage(2, 4), SearchStage(2, 1)), block_sizes=(8,))
    g = fme.estimate_motion(fr[2], fr[1], small)
    std = fme.estimate_motion(fr[3], fr[2], fme.get_preset("standard"))
    labels = synth.block_labels(256, 256, 4)
    res = pipeline.run_sequence(fr, dict(enumerate(labels)),
                                PipelineConfig(fme=c1, refine_enabled=True, max_gop=4, aem_threshold=float("inf")))
    print("stage", int(f[0].candidate_evals), "small", int(g[0].candidate_evals),
          "std", [int(x.candidate_evals) for x in std], "keys", res.keyframes,
          "labels", int(np.asarray(res.labels[-1].classes, np.int64).sum()))


if __name__ == "__main__":
    main()
