import sys, numpy as np
sys.path.insert(0, '.')
which = sys.argv[1]
from paper_2508_05990_b200 import fme, mv_refine, propagate, frame_select as fs
rng = np.random.default_rng(9)
if which == "energy":
    a, b = rng.random((64, 64)), rng.random((64, 64))
    print(fme.block_energy(a, b, 0.1))
elif which == "refine":
    mv = np.zeros((3, 3, 2), np.int64); mv[..., 0] = 2; mv[1, 1] = (30, -12)
    f = fme.MotionField(16, 3, 3, mv, np.zeros((3, 3)), np.ones((3, 3), bool))
    print(mv_refine.refine_mvs(f, 4).mv[..., 0])
elif which == "decide":
    _, st = fs.open_gop(0, 2, 2, 16)
    e = np.full((2, 2), 0.4)
    field = fme.MotionField(16, 2, 2, np.zeros((2, 2, 2), np.int64), e, np.ones((2, 2), bool))
    print(fs.decide(st, field, 1, aem_threshold=1.0))
elif which == "predict":
    from paper_2508_05990_b200.frame_io import LabelMap
    mv = rng.integers(-20, 21, (4, 4, 2)).astype(np.int64)
    field = fme.MotionField(8, 4, 4, mv, np.zeros((4, 4)), np.ones((4, 4), bool))
    cls = rng.integers(0, 7, (60, 50)).astype(np.uint8)
    print(propagate.predict_labels(LabelMap(50, 60, cls, 7), field, 2).classes.sum())
