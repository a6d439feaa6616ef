import numpy as np, sys, subprocess
sys.path.insert(0, '.')
if len(sys.argv) == 1:
    for args in ["16 3 0 bayer", "14 3 0 bayer", "14 3 1 bayer", "16 3 1 bayer", "14 3 0 luma", "13 3 0 luma", "16 5 0 bayer"]:
        r = subprocess.run([sys.executable, __file__] + args.split(), capture_output=True, text=True)
        print(args, "->", (r.stdout.strip().splitlines() or ["?"])[-1], "ERR" if r.returncode else "")
    sys.exit(0)
from paper_2508_05990_b200 import fme
from paper_2508_05990_b200.frame_io import Frame, FrameKind
ox, oy, rg, kind = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
k = FrameKind.BAYER_RGGB if kind == "bayer" else FrameKind.LUMA
rng = np.random.default_rng(5)
a = rng.integers(0, 256, (96, 80)).astype(np.uint8); b = rng.integers(0, 256, (96, 80)).astype(np.uint8)
cur, ref = Frame(80, 96, a, k), Frame(80, 96, b, k)
print(fme.search_stage(cur, ref, (ox, oy), 16, (-3, 3), rg, 1, fme.FmeConfig()))
