import sys, os, numpy as np, subprocess
sys.path.insert(0, '.')
if len(sys.argv) == 1:
    cases = ["4,8 0,1 0,1", "2,4 0,1 0,1", "2,4 2,4 0,1", "4,8 4,8 0,1", "4,8 2,4 0,1", "1,1 1,1 0,1", "4,8 2,4 2,1"]
    for c in cases:
        for env in ({}, {"BMC_NO_TMA": "1"}):
            r = subprocess.run([sys.executable, __file__] + c.split(), capture_output=True, text=True,
                               env={**os.environ, "BMC_SYNC_DEBUG": "1", **env})
            print(c, env, "->", (r.stdout.strip().splitlines() or ["?"])[-1], "|", (r.stderr.strip().splitlines() or [""])[-1][:200])
    sys.exit(0)
from paper_2508_05990_b200 import fme
from paper_2508_05990_b200.fme import FmeConfig, SearchStage
from paper_2508_05990_b200.frame_io import Frame, FrameKind
from oracle import bayermc_oracle as O
st = [tuple(int(v) for v in s.split(",")) for s in sys.argv[1:4]]
cfg = FmeConfig(stages=tuple(SearchStage(*s) for s in st), block_sizes=(64,))
rng = np.random.default_rng(1)
a = rng.integers(0, 256, (256, 256)).astype(np.uint8); b = rng.integers(0, 256, (256, 256)).astype(np.uint8)
out = fme.estimate_motion(Frame(256, 256, a, FrameKind.BAYER_RGGB), Frame(256, 256, b, FrameKind.BAYER_RGGB), cfg)
want = O.estimate_motion(O.search_planes(a, True), O.search_planes(b, True), O.cfg_dict(stages=st, block_sizes=(64,)))
print("ok", out[0].candidate_evals, bool(np.array_equal(out[0].mv, want[0].mv) and np.array_equal(out[0].energy, want[0].energy)))
