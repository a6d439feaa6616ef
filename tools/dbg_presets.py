import sys, os, numpy as np, subprocess
sys.path.insert(0, '.')
if len(sys.argv) == 1:
    for args in ["standard 128 128", "standard 256 256", "mode3 128 128", "mode4 256 192", "mode5 192 256"]:
        r = subprocess.run([sys.executable, __file__] + args.split(), capture_output=True, text=True,
                           env={**os.environ, "BMC_SYNC_DEBUG": "1"})
        print(args, "->", (r.stdout.strip().splitlines() or ["?"])[-1], "|", (r.stderr.strip().splitlines() or [""])[-1][:400])
    sys.exit(0)
from paper_2508_05990_b200 import fme
from paper_2508_05990_b200.frame_io import Frame, FrameKind
name, h, w = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
rng = np.random.default_rng(1)
a = rng.integers(0, 256, (h, w)).astype(np.uint8); b = rng.integers(0, 256, (h, w)).astype(np.uint8)
out = fme.estimate_motion(Frame(w, h, a, FrameKind.BAYER_RGGB), Frame(w, h, b, FrameKind.BAYER_RGGB), fme.get_preset(name))
print("ok", [f.candidate_evals for f in out])
