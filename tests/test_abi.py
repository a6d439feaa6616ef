"""CPU: the C-ABI library builds/loads, exports every symbol include/*.h
declares, and its host-only entry points validate arguments like the
reference (no GPU compute is called here)."""

import ctypes
import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def header_symbols():
    txt = "\n".join(h.read_text() for h in sorted((ROOT / "include").glob("*.h")))
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(bmc_[a-z_0-9]+)\s*\(", txt, re.M)))


def test_library_exports_every_header_symbol():
    from paper_2508_05990_b200 import _native as N
    lib = N.load()
    syms = header_symbols()
    assert len(syms) >= 12
    for s in syms:
        assert hasattr(lib, s), s
    out = subprocess.run(["nm", "-D", "--defined-only", str(N.lib_path())], capture_output=True, text=True).stdout
    for s in syms:
        assert re.search(rf"\bT {s}\b", out), f"{s} not exported"
    assert set(N.EXPORTED_SYMBOLS) == set(syms)


def test_library_is_sm100a_only():
    from paper_2508_05990_b200 import _native as N
    out = subprocess.run(["cuobjdump", "--list-elf", str(N.lib_path())], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)
    sass = subprocess.run(["cuobjdump", "-sass", str(N.lib_path())], capture_output=True, text=True).stdout
    assert "VABSDIFF4.U8.ACC" in sass  # packed uint8 SAD
    assert "VIMNMX.U16x2" in sass  # packed uint16 path
    assert "UTMALDG" in sass  # TMA window staging


def test_fill_params_geometry_and_validation():
    from paper_2508_05990_b200 import _native as N
    from paper_2508_05990_b200.fme import FmeConfig, SearchStage
    p = N.make_params(N.KIND_BAYER, 1, 1080, 1920, FmeConfig(stages=(SearchStage(16, 1), SearchStage(0, 1),
                                                                     SearchStage(0, 1)), block_sizes=(16,)))
    assert (p.planes, p.real_h, p.real_w, p.pad_h, p.pad_w) == (4, 540, 960, 544, 960)
    assert p.pitch % 16 == 0 and p.plane_stride == p.pad_h * p.pitch and p.frame_stride == 4 * p.plane_stride
    assert p.one_minus_lam == 1.0 - 0.1
    p2 = N.make_params(N.KIND_LUMA, 2, 70, 54, FmeConfig())
    assert (p2.planes, p2.max_value, p2.pad_h, p2.pad_w) == (1, 65535, 128, 64)

    class Bad:
        stages = (SearchStage(1, 1),) * 3
        lam = 0.1
        sparsity_tolerance = 0.03
        split_threshold = 0.02
        refine_block_threshold = 0.05

    for sizes, msg in [((12,), "power of two"), ((64, 16), "halve"), ((128,), "64-sample maximum")]:
        Bad.block_sizes = sizes
        with pytest.raises(ValueError, match=msg):
            N.make_params(N.KIND_LUMA, 1, 64, 64, Bad)
    Bad.block_sizes = (16,)
    with pytest.raises(ValueError, match="even width and height"):
        N.make_params(N.KIND_BAYER, 1, 63, 64, Bad)


def test_error_string_and_status_mapping():
    from paper_2508_05990_b200 import _native as N
    lib = N.load()
    assert lib.bmc_version().startswith(b"bmc_b200")
    # argument errors surface as ValueError with the C message (no CUDA needed)
    rc = lib.bmc_refine_mvs(None, None, 1, 0, 4, 16, 4, None, None, None, None, None, None, None, None)
    with pytest.raises(ValueError, match="empty motion field"):
        N.check(rc)
    rc = lib.bmc_predict_labels(ctypes.c_void_p(8), 0, 0, None, 1, 1, None, None, 0, 0, 100, 100, ctypes.c_void_p(8),
                                0, 0, 1, 1, 16, 3, None)
    with pytest.raises(ValueError, match="scale must be 1 or 2"):
        N.check(rc)


def test_build_entry_point_compiles_for_sm100a(tmp_path):
    """__graft_entry__.build() path: nvcc cross-compiles here without a GPU."""
    from paper_2508_05990_b200 import build as B
    assert "arch=compute_100a,code=sm_100a" in " ".join(B.ARCH)
    assert B.LIB.exists()
