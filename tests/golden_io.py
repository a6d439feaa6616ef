"""Load the reference-generated golden fixtures (tests/golden/*.npz)."""

from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"


def load(name):
    return dict(np.load(GOLDEN / name, allow_pickle=False))


def me_fixture_names():
    return sorted(p.name for p in GOLDEN.glob("me_*.npz"))


def pipe_fixture_names():
    return sorted(p.name for p in GOLDEN.glob("pipe_*.npz"))


def pipe_inputs(d):
    if "clip" in d:
        return d["clip"], d["key_labels"]
    base = load(str(d["inputs_from"]))
    return base["clip"], base["key_labels"]


def oracle_cfg(d):
    from oracle import bayermc_oracle as O
    return O.cfg_dict(stages=[tuple(int(v) for v in s) for s in d["stages"]], lam=float(d["lam"]),
                      block_sizes=tuple(int(b) for b in d["block_sizes"]), split_threshold=float(d["split"]),
                      sparsity_tolerance=float(d["tol"]), refine_block_threshold=float(d["refine_thr"]))


def fme_config(d):
    from paper_2508_05990_b200.fme import FmeConfig, SearchStage
    return FmeConfig(stages=tuple(SearchStage(int(r), int(s)) for r, s in d["stages"]), lam=float(d["lam"]),
                     block_sizes=tuple(int(b) for b in d["block_sizes"]), split_threshold=float(d["split"]),
                     sparsity_tolerance=float(d["tol"]), refine_block_threshold=float(d["refine_thr"]))


def levels(d):
    return [(d[f"L{i}_mv"], d[f"L{i}_energy"], d[f"L{i}_matched"], int(d[f"L{i}_evals"]), int(d[f"L{i}_block"]))
            for i in range(int(d["levels"]))]


def pipeline_config(d):
    from paper_2508_05990_b200.config import PipelineConfig
    return PipelineConfig(fme=fme_config(d), refine_enabled=bool(d.get("refine", False)), aem_threshold=float(d["aem"]),
                          max_gop=int(d["max_gop"]) if bool(d["has_max_gop"]) else None,
                          aem_statistic=str(d["statistic"]), reference_policy=str(d["policy"]))
