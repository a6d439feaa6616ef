"""B200-native temporal-redundancy back end of arXiv 2508.05990 (ISP-less
Bayer video vision): block-matching ME on raw Bayer frames, MV refinement,
motion compensation, the CaBR block mask and AEM key-frame selection.

The modules mirror the reference package ``bayermc`` (fme, mv_refine,
propagate, frame_select, frame_io, config, pipeline) with identical
signatures; the arithmetic runs in hand-written sm_100a kernels
(``csrc/``) behind the C ABI in ``include/bmc.h``.
"""

from . import config, engine, fme, frame_io, frame_select, metrics, mv_refine, pipeline, propagate, synth  # noqa: F401
from ._native import load as load_library  # noqa: F401

__version__ = "0.1.0"
